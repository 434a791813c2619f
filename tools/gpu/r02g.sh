out=gpurun_out/r02h; mkdir -p $out
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > $out/make.log 2>&1; echo make=$?
TINV_A2=0 TINV_DBG=1 timeout 600 python tools/phase_window.py cfg4 3950:4050 > $out/phase_dbg1.txt 2>&1; echo phase=$?
make -s -C paper_1209_1910_b200/csrc -B > /dev/null 2>&1

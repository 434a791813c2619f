out=gpurun_out/r02p; mkdir -p $out
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > $out/make.log 2>&1; echo make=$?
TINV_LAB=8 TINV_DBG=4 timeout 600 python tools/phase_window.py cfg4 3950:4050 > $out/phase_lab.txt 2>&1; echo phase=$?
make -s -C paper_1209_1910_b200/csrc -B > /dev/null 2>&1
cat $out/phase_lab.txt

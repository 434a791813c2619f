out=gpurun_out/r02t; mkdir -p $out
timeout 600 tools/micro/fp64_peak > $out/fp64_peak.txt 2>&1; echo fp64=$?
timeout 900 python tools/a2_sweep.py cfg4 "TINV_PF=0" "TINV_PF=16" "TINV_PF=32" > $out/pf.txt 2>&1; echo pf=$?
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > $out/make.log 2>&1; echo make=$?
TINV_DBG=8 timeout 600 python tools/phase_window.py cfg4 3950:4050 > $out/phase_sweep.txt 2>&1; echo phase=$?
make -s -C paper_1209_1910_b200/csrc -B > /dev/null 2>&1
cat $out/*.txt

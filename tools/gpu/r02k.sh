out=gpurun_out/r02k; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3 or scaled_configs or row_split or restart or cfg4_giant" > $out/pytest.log 2>&1; echo pytest=$?; tail -3 $out/pytest.log
timeout 900 python tools/a2_sweep.py cfg4 "TINV_A2=1" "TINV_A2=0" > $out/a2.txt 2>&1; echo a2=$?
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > $out/make.log 2>&1; echo make=$?
TINV_A2=0 TINV_DBG=2 timeout 600 python tools/phase_window.py cfg4 3950:4050 > $out/phase_dbg2.txt 2>&1; echo phase=$?
make -s -C paper_1209_1910_b200/csrc -B > /dev/null 2>&1
cat $out/a2.txt $out/phase_dbg2.txt

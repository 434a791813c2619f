out=gpurun_out/r02u; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "lookahead or cfg4_giant" > $out/pytest.log 2>&1; echo pytest=$?; tail -2 $out/pytest.log
timeout 900 python tools/a2_sweep.py cfg4 "TINV_LAB=8" "TINV_LAB=0" > $out/lab.txt 2>&1; echo lab=$?
cat $out/lab.txt

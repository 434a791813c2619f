out=gpurun_out/r02r; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "row_split or scaled_configs or cfg3 or cfg2 or lookahead or mgs or ordinary" > $out/pytest.log 2>&1; echo pytest=$?; tail -5 $out/pytest.log

out=gpurun_out/r02m; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "mgs or ordinary or reorth or restart" --durations=10 > $out/pytest.log 2>&1; echo pytest=$?; tail -15 $out/pytest.log

out=gpurun_out/r02q; mkdir -p $out
timeout 600 python -m pytest tests/test_multirank_gpu.py -x -q > $out/pytest_ipc.log 2>&1; echo ipc=$?; tail -15 $out/pytest_ipc.log
timeout 2400 python -m pytest tests -m gpu -x -q --durations=12 > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -16 $out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --no-cpu-baseline > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo bench4=$?
python tools/bench_brief.py $out/bench_cfg4.json

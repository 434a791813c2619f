# Quick GPU iteration: parity tests, then short benches of the given configs.
set -x
mkdir -p gpurun_out
timeout ${PT_TIMEOUT:-900} python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for c in ${CFGS:-cfg2 cfg3 cfg4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-5} --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?
  python tools/bench_brief.py gpurun_out/bench_$c.json
done

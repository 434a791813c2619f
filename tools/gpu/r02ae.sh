# Column-form TN (TINV_TNC): full GPU suite (defaults), cfg4 / cfg5 with TNC on / off, cfg4 A2C on / off.
set -x
out=gpurun_out/r02ae; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
for v in "TINV_TNC=1" "TINV_TNC=0" "TINV_A2C=0"; do
env $v timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > "$out/bench_cfg4_$v.json" 2> /dev/null; echo b4=$?
echo $v; python tools/bench_brief.py "$out/bench_cfg4_$v.json"
done
for v in "TINV_TNC=1" "TINV_TNC=0"; do
env $v timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > "$out/bench_cfg5_$v.json" 2> /dev/null; echo b5=$?
echo $v; python tools/bench_brief.py "$out/bench_cfg5_$v.json"
done

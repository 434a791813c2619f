# Column-owner A2 (TINV_A2C) and the non-inlined sweep chunk (TINV_SWEEP2=2): GPU suite, benches.
set -x
out=gpurun_out/r02ab; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo b5=$?
python tools/bench_brief.py $out/bench_cfg5.json
for v in "TINV_A2C=1" "TINV_A2C=0" "TINV_SWEEP2=2"; do
env $v timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg4_$v.json 2> $out/bench_cfg4_$v.err; echo b4=$?
echo $v; python tools/bench_brief.py $out/bench_cfg4_$v.json
done
TINV_SWEEP2=2 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg5_sw2.json 2> $out/bench_cfg5_sw2.err; echo b5=$?
python tools/bench_brief.py $out/bench_cfg5_sw2.json

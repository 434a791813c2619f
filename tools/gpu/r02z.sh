# Two-thread back sweep (TINV_SWEEP2): GPU suite, then cfg5/cfg4 with it on and off.
set -x
out=gpurun_out/r02z; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
for sw in 1 0; do
TINV_SWEEP2=$sw timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg5_sw$sw.json 2> $out/bench_cfg5_sw$sw.err; echo b5=$?
python tools/bench_brief.py $out/bench_cfg5_sw$sw.json
TINV_SWEEP2=$sw timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg4_sw$sw.json 2> $out/bench_cfg4_sw$sw.err; echo b4=$?
python tools/bench_brief.py $out/bench_cfg4_sw$sw.json
done

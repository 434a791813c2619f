# Same-box A/B: TINV_TYR (T_p yrow kept) and TINV_A2C (parallel block table), cfg4 x4, cfg5 x2.
set -x
out=gpurun_out/r02ag; mkdir -p $out
timeout 300 python -m pytest tests -m gpu -x -q -k "lookahead or scaled_configs" > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $out/pytest_gpu.log
for v in "TINV_TYR=1 TINV_A2C=1" "TINV_TYR=0 TINV_A2C=1" "TINV_TYR=1 TINV_A2C=0" "TINV_TYR=0 TINV_A2C=0"; do
env $v timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > "$out/bench_cfg4_$v.json" 2> /dev/null; echo b4=$?
echo $v; python tools/bench_brief.py "$out/bench_cfg4_$v.json"
done
for v in "TINV_TYR=1" "TINV_TYR=0"; do
env $v timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > "$out/bench_cfg5_$v.json" 2> /dev/null; echo b5=$?
echo $v; python tools/bench_brief.py "$out/bench_cfg5_$v.json"
done

# Evidence at HEAD a253e19 (column-owner A2, T_p yrow reuse, fused in-block dots): GPU suite, smoke, default bench (cfg5), cfg4 bench.
set -x
out=gpurun_out/r02ba; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo smoke=$?; cat $out/smoke.log
timeout 1200 python bench.py > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo bench5=$?
timeout 900 python bench.py --config cfg4 --no-cpu-baseline > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo bench4=$?
for c in cfg4 cfg5; do python tools/bench_brief.py $out/bench_$c.json; done

# Re-entry check: full GPU parity suite, cfg4 bench (default), cfg2/cfg5 benches, A2 knob sweep.
set -x
out=gpurun_out/r02c; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --no-cpu-baseline > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo bench4=$?
timeout 600 python tools/a2_sweep.py cfg4 "TINV_A2=0" "TINV_A2=1" "TINV_A2=1,TINV_BANDCH=8" "TINV_A2=1,TINV_POLLNS=200" > $out/a2.txt 2>&1; echo a2=$?
timeout 600 python bench.py --config cfg2 --steps 10 --no-cpu-baseline > $out/bench_cfg2.json 2> $out/bench_cfg2.err; echo bench2=$?
timeout 600 python bench.py --config cfg3 --steps 3 --no-cpu-baseline > $out/bench_cfg3.json 2> $out/bench_cfg3.err; echo bench3=$?
timeout 900 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo bench5=$?
for c in cfg2 cfg3 cfg4 cfg5; do python tools/bench_brief.py $out/bench_$c.json; done

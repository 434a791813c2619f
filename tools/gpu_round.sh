# One GPU session for the round's evidence: smoke, parity tests, benches (cfg2 default with
# the CPU baseline, then cfg1/3/4/5), the reference arm, launch list and ncu full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref_cfg2.json 2> gpurun_out/bench_ref_cfg2.err; echo ref=$?
for c in cfg1 cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; done
timeout 900 python bench.py --config cfg5 --steps 1 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench_cfg5=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
# the resident cWY launches of one step (three thread-block-cluster groups on cfg2)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resident -s 9 -c 3 -o gpurun_out/prof_cwy_cfg2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched -s 3 -c 1 -o gpurun_out/prof_batched_cfg2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full2.log 2>&1; echo ncu_full2=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cwy -c 1 -o gpurun_out/prof_cwy_cfg3 -f python tools/run_case.py --config cfg3 --reps 1 > gpurun_out/ncu_full3.log 2>&1; echo ncu_full3=$?
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python tools/bench_brief.py gpurun_out/bench_$c.json; done

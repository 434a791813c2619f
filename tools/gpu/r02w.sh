# Evidence round r02w: default bench = cfg5; full GPU suite; reference arm; launch list; ncu full of cfg5.
set -x
out=gpurun_out/r02w; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 $out/pytest_gpu.log
timeout 1200 python bench.py > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 > $out/bench_ref_cfg5.json 2> $out/bench_ref_cfg5.err; echo ref=$?
timeout 900 python bench.py --config cfg4 --no-cpu-baseline > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo bench4=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_cfg5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:cwy_kernel -c 1 -f -o $out/prof_cwy_cfg5 python tools/run_case.py --config cfg5 --reps 1 > $out/ncu_full.log 2>&1; echo ncu_full=$?
ncu -i $out/prof_cwy_cfg5.ncu-rep --page raw --csv > $out/prof_cwy_cfg5_raw.csv 2>/dev/null; echo raw=$?
for c in cfg4 cfg5; do python tools/bench_brief.py $out/bench_$c.json; done

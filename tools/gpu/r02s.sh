# Evidence round r02s: smoke, default bench (cfg4) with CPU baseline, reference arm, benches of
# cfg2/cfg3/cfg5, launch list of the bench, ncu --set full of one cfg4 cwy_kernel launch.
set -x
out=gpurun_out/r02s; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 > $out/bench_ref_cfg4.json 2> $out/bench_ref_cfg4.err; echo ref=$?
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > $out/bench_cfg2.json 2> $out/bench_cfg2.err; echo bench2=$?
timeout 600 python bench.py --config cfg3 --steps 5 --no-cpu-baseline > $out/bench_cfg3.json 2> $out/bench_cfg3.err; echo bench3=$?
timeout 1200 python bench.py --config cfg5 --steps 2 --no-cpu-baseline > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo bench5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_cfg4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cwy_kernel -c 1 -f -o $out/prof_cwy_cfg4 python tools/run_case.py --config cfg4 --reps 1 > $out/ncu_full.log 2>&1; echo ncu_full=$?
ncu -i $out/prof_cwy_cfg4.ncu-rep --page raw --csv > $out/prof_cwy_cfg4_raw.csv 2>/dev/null; echo raw=$?
for c in cfg2 cfg3 cfg4 cfg5; do python tools/bench_brief.py $out/bench_$c.json; done

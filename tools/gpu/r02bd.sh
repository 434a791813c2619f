# Final evidence of round 2 (build with the early staging-buffer release, CTA-0 share of pass D,
# band size): smoke, the GPU suite, default bench (cfg5, full contract), the reference arm,
# cfg2/cfg3/cfg4 benches, the bench's ncu launch list, DRAM bytes of the cfg5 cWY interval,
# ncu --set full of one cfg4 cwy_kernel launch.
set -x
out=gpurun_out/r02bd; mkdir -p $out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo smoke=$?; cat $out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 $out/pytest_gpu.log
timeout 1500 python bench.py > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo bench5=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_cfg5.json 2> $out/bench_ref_cfg5.err; echo ref=$?
for c in cfg2 cfg3 cfg4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err; echo bench_$c=$?; done
for c in cfg5 cfg2 cfg3 cfg4; do python tools/bench_brief.py $out/bench_$c.json; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_cfg5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'cwy_kernel|dz_' -c 3 --csv --log-file $out/dram_cfg5.csv python tools/run_case.py --config cfg5 --reps 1 > $out/ncu_dram5.log 2>&1; echo ncu_dram5=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'cwy_kernel|dz_gemm' -c 2 -f -o $out/prof_cfg4 python tools/run_case.py --config cfg4 --reps 1 > $out/ncu_full.log 2>&1; echo ncu_full=$?
ncu -i $out/prof_cfg4.ncu-rep --page raw --csv > $out/prof_cfg4_raw.csv 2>/dev/null; echo raw=$?
python tools/ncu_summary.py $out/launches_cfg5.csv > $out/launches_cfg5.txt 2>&1; cat $out/launches_cfg5.txt | head -20
cat $out/dram_cfg5.csv | tail -12

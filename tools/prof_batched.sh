set -x
CFG=${CFG:-cfg2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched -s 3 -c 1 -f -o gpurun_out/prof_batched_$CFG python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_batched_$CFG.log 2>&1
echo ncu=$?

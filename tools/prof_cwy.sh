# ncu --set full capture of the cWY kernel on one config (after a plain run exits 0)
set -x
CFG=${CFG:-cfg2}
python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_plain_$CFG.json 2> gpurun_out/prof_plain_$CFG.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cwy -s 3 -c 1 -f -o gpurun_out/prof_cwy_$CFG python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cwy_$CFG.log 2>&1
echo ncu=$?

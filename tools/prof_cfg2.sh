set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:cwy -s 3 -c 1 -o gpurun_out/prof_cwy_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:batched -s 3 -c 1 -o gpurun_out/prof_batched_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo ncu3=$?

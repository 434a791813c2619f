python tools/run_case.py --config cfg4 --n 2000 --reps 2 --profile > gpurun_out/rc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cwy -s 1 -c 1 -o gpurun_out/prof_cwy_cfg4n2000 python tools/run_case.py --config cfg4 --n 2000 --reps 2 > gpurun_out/ncu_cwy.log 2>&1
echo ncu=$?
tail -3 gpurun_out/rc_plain.log

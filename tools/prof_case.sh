# ncu --set full of the cWY kernel on a (scaled) config via run_case.py (after a plain run)
set -x
CFG=${CFG:-cfg4}; N=${N:-3000}
timeout 300 python tools/run_case.py --config $CFG --n $N --reps 2 > gpurun_out/rc_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cwy -s 1 -c 1 -f -o gpurun_out/prof_cwy_${CFG}_$N python tools/run_case.py --config $CFG --n $N --reps 2 > gpurun_out/ncu_case.log 2>&1
echo ncu=$?

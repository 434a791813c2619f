# per-launch durations (ncu launch list) of one tinv_eigvecs call on a config
CFG=${CFG:-cfg2}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_case.csv python tools/run_case.py --config $CFG --reps 2 ${N:+--n $N} > gpurun_out/launches_case.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_case.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size'); bi=h.index('Block Size')
for r in rows[1:]: print(r[ki][:60], r[gi], r[bi], float(r[vi].replace(',',''))/1e3, 'us')
PY

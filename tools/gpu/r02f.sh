# SASS-level source counters of the wide kernel on cfg4 (n = 4000)
out=gpurun_out/r02f; mkdir -p $out
timeout 1200 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none -k regex:cwy_kernel -c 1 -f -o $out/src4000 python tools/run_case.py --config cfg4 --n 4000 --reps 1 > $out/ncu.log 2>&1; echo ncu=$?
ncu -i $out/src4000.ncu-rep --page source --csv --print-source sass > $out/src_sass.csv 2>/dev/null; echo exp=$?
ls -la $out

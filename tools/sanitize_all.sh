#!/bin/bash
# compute-sanitizer over the product kernels (libtinv.so) on small cases; summaries -> $1/
out=${1:-gpurun_out/sanitize}
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for c in cfg1 cfg2 cfg4s vr2 cfg3s mgs; do
    timeout 900 $CS --tool $tool --kernel-name regex:'(prep|batched|pack|finalize|cwy|bisect)' \
      --print-limit 20 --error-exitcode 9 python tools/sanitize_case.py $c > $out/${tool}_$c.log 2>&1
    echo "$tool $c rc=$?" | tee -a $out/summary.txt
  done
done

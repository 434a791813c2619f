# Same-box build A/B: libtinv_ref.so (commit 2e119d5) vs the working build; cfg4 alternating, cfg5 each; chain micro.
set -x
out=gpurun_out/r02aj; mkdir -p $out
(cd tools/micro && ./sweep_floor) > $out/sweep_floor.txt 2>&1; cat $out/sweep_floor.txt
for i in 1 2; do for lib in ref cur; do
  if [ $lib = ref ]; then export TINV_LIB_VARIANT=ref; else unset TINV_LIB_VARIANT; fi
  timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > "$out/bench_cfg4_${lib}_$i.json" 2> /dev/null; echo b4=$?
  echo "$lib $i"; python tools/bench_brief.py "$out/bench_cfg4_${lib}_$i.json"
done; done
for lib in ref cur; do
  if [ $lib = ref ]; then export TINV_LIB_VARIANT=ref; else unset TINV_LIB_VARIANT; fi
  timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > "$out/bench_cfg5_${lib}.json" 2> /dev/null; echo b5=$?
  echo "$lib"; python tools/bench_brief.py "$out/bench_cfg5_${lib}.json"
done

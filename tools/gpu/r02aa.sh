# Streamed BL1 (TINV_BL1): GPU suite, cfg5 / cfg4 benches (BL1 on / off), back-sweep chain floor micro.
set -x
out=gpurun_out/r02aa; mkdir -p $out
(cd tools/micro && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o sweep_floor sweep_floor.cu && ./sweep_floor) > $out/sweep_floor.txt 2>&1; cat $out/sweep_floor.txt
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo b5=$?
python tools/bench_brief.py $out/bench_cfg5.json
for b in 1 0; do
TINV_BL1=$b timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg4_bl$b.json 2> $out/bench_cfg4_bl$b.err; echo b4=$?
python tools/bench_brief.py $out/bench_cfg4_bl$b.json
done

# A2C R1 with batched loads; ws_pass micro (colacc / rowdots one / two vectors); cfg4 A2C on/off, band sizes.
set -x
out=gpurun_out/r02ac; mkdir -p $out
(cd tools/micro && nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ws_pass ws_pass.cu 2>/dev/null && ./ws_pass) > $out/ws_pass.txt 2>&1; cat $out/ws_pass.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "lookahead or cfg4 or cfg5 or scaled or virtual" > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
for v in "TINV_A2C=1" "TINV_A2C=0" "TINV_A2C=1 TINV_BANDCH=4" "TINV_A2C=1 TINV_BANDCH=16"; do
env $v timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > "$out/bench_cfg4_$v.json" 2> /dev/null; echo b4=$?
echo $v; python tools/bench_brief.py "$out/bench_cfg4_$v.json"
done
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo b5=$?
python tools/bench_brief.py $out/bench_cfg5.json

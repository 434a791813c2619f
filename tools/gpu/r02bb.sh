# Deferred final pass D (dz.cu): targeted tests, GPU suite, cfg4 / cfg5 benches (deferral on / off).
set -x
out=gpurun_out/r02bb; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -k deferred -x -q > $out/pytest_dz.log 2>&1; rc=$?; echo pytest_dz=$rc; tail -30 $out/pytest_dz.log
[ $rc = 0 ] || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
timeout 900 python bench.py --config cfg4 --steps 3 --no-cpu-baseline --no-e2e > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo bench4=$?
TINV_DZ=0 timeout 900 python bench.py --config cfg4 --steps 3 --no-cpu-baseline --no-e2e > $out/bench_cfg4_nodz.json 2> $out/bench_cfg4_nodz.err; echo bench4n=$?
timeout 1200 python bench.py --steps 3 --no-cpu-baseline --no-e2e > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo bench5=$?
timeout 600 python bench.py --config cfg3 --steps 5 --no-cpu-baseline --no-e2e > $out/bench_cfg3.json 2> $out/bench_cfg3.err; echo bench3=$?
for c in cfg4 cfg4_nodz cfg5 cfg3; do echo $c; python tools/bench_brief.py $out/bench_$c.json; done

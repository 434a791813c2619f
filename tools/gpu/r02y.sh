# A2 block-end prefetch: GPU suite, cfg5/cfg4 bench, then the debug build's GEMM sub-timers and per-CTA busy times.
set -x
out=gpurun_out/r02y; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg5.json 2> $out/bench_cfg5.err; echo b5=$?
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo b4=$?
python tools/bench_brief.py $out/bench_cfg5.json; python tools/bench_brief.py $out/bench_cfg4.json
make -C paper_1209_1910_b200/csrc -B -j8 EXTRA=-DTINV_WIDE_DEBUG > $out/build.log 2>&1; echo build=$?
TINV_DBG=16 TINV_PROF_CTA=1 timeout 600 python tools/phase_window.py cfg5 8000:8040 14000:14040 > $out/pw.txt 2>&1; echo pw=$?
cat $out/pw.txt

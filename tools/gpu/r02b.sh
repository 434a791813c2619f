set -x
mkdir -p gpurun_out/r02b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02b/smi.txt 2>&1
timeout 600 python bench.py --steps 3 > gpurun_out/r02b/bench_cfg4.json 2> gpurun_out/r02b/bench_cfg4.err; echo bench=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "restart or maxits or scaled or sign_rule or cfg1" > gpurun_out/r02b/pytest_new.log 2>&1; echo pytest=$?
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > /dev/null 2>&1; echo make=$?
TINV_PROF_CTA=1 timeout 600 python tools/phase_window.py cfg4 500:600 3950:4050 7400:7500 > gpurun_out/r02b/phase_cfg4.txt 2>&1; echo phase=$?

# Usage: bash tools/gpu/measure.sh TAG [pytest -k expr]
# cfg4 bench (product build), a pytest subset, then the debug build's phase windows.
tag=$1; kexpr=${2:-}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
if [ -n "$kexpr" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$kexpr" > $out/pytest.log 2>&1; echo pytest=$?
fi
timeout 600 python bench.py --steps 3 --no-cpu-baseline > $out/bench_cfg4.json 2> $out/bench_cfg4.err; echo bench=$?
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > /dev/null 2>&1; echo make=$?
TINV_PROF_CTA=1 timeout 600 python tools/phase_window.py cfg4 500:600 3950:4050 7400:7500 > $out/phase_cfg4.txt 2>&1; echo phase=$?
make -s -C paper_1209_1910_b200/csrc -B > /dev/null 2>&1

# Diagnosis of the cfg5 default: per-window phase costs, per-CTA busy times, back-sweep parts (debug build).
set -x
out=gpurun_out/r02x; mkdir -p $out
make -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > $out/build.log 2>&1; echo build=$?
TINV_PROF_CTA=1 timeout 600 python tools/phase_window.py cfg5 2000:2040 8000:8040 14000:14040 > $out/pw_cta.txt 2>&1; echo pw=$?
TINV_DBG=8 timeout 600 python tools/phase_window.py cfg5 8000:8040 > $out/pw_sweep.txt 2>&1; echo pws=$?
cat $out/pw_cta.txt $out/pw_sweep.txt

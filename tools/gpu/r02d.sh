# Phase windows (debug build, per-CTA busy times) for A2 off/on; A2 knob sweep.
out=gpurun_out/r02d; mkdir -p $out
timeout 900 python tools/a2_sweep.py cfg4 "TINV_A2=0" "TINV_A2=1,TINV_BANDCH=8" "TINV_A2=1,TINV_BANDCH=16" "TINV_A2=1,TINV_BANDCH=32" "TINV_A2=0" > $out/a2.txt 2>&1; echo a2=$?
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > /dev/null 2>&1; echo make=$?
TINV_A2=0 TINV_PROF_CTA=1 timeout 600 python tools/phase_window.py cfg4 500:600 3950:4050 7400:7500 > $out/phase_cfg4_a20.txt 2>&1; echo phase=$?
TINV_A2=1 TINV_BANDCH=16 TINV_PROF_CTA=1 timeout 600 python tools/phase_window.py cfg4 3950:4050 > $out/phase_cfg4_a21.txt 2>&1; echo phase=$?
make -s -C paper_1209_1910_b200/csrc -B > /dev/null 2>&1

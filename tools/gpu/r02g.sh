out=gpurun_out/r02j; mkdir -p $out
make -s -C paper_1209_1910_b200/csrc -B EXTRA=-DTINV_WIDE_DEBUG > $out/make.log 2>&1; echo make=$?
for n in 2000 8000; do
TINV_A2=0 TINV_DBG=2 PW_N=$n timeout 600 python tools/phase_window.py cfg4 $((n/2-50)):$((n/2+50)) > $out/phase_dbg2_$n.txt 2>&1; echo phase=$?
done
make -s -C paper_1209_1910_b200/csrc -B > /dev/null 2>&1

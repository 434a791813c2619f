out=gpurun_out/r02v; mkdir -p $out
timeout 1500 python tools/a2_sweep.py cfg4 "TINV_BANDCH=16" "TINV_BANDCH=8" "TINV_BANDCH=32" "TINV_PIECE_COST=2500" "TINV_PIECE_COST=6000" "TINV_LAB=4" "TINV_A2=0" > $out/knobs.txt 2>&1; echo k=$?
cat $out/knobs.txt

out=gpurun_out/$1; mkdir -p $out
timeout 900 python tools/a2_sweep.py cfg4 "TINV_A2=0" "TINV_A2=1" "TINV_A2=1,TINV_POLLNS=200" "TINV_A2=1,TINV_BANDCH=8" "TINV_A2=1,TINV_BANDCH=16" "TINV_A2=1,TINV_BANDCH=2,TINV_POLLNS=100" > $out/a2.txt 2>&1; echo a2=$?

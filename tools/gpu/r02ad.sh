# Bisect the illegal address of r02ac: one failing test under knob combinations (separate processes).
set -x
out=gpurun_out/r02ad; mkdir -p $out
for v in "TINV_SWEEP2=1 TINV_A2C=1 TINV_TNC=0" "TINV_SWEEP2=2 TINV_A2C=0 TINV_TNC=0" "TINV_SWEEP2=2 TINV_A2C=1 TINV_TNC=0" "TINV_SWEEP2=1 TINV_A2C=0 TINV_TNC=1" "TINV_SWEEP2=1 TINV_A2C=1 TINV_TNC=1"; do
  echo "== $v"
  env $v timeout 300 python -m pytest tests -m gpu -x -q -k "test_scaled_configs_full or lookahead_parity" 2>&1 | tail -2
done
(cd tools/micro && nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ws_pass ws_pass.cu 2>/dev/null && ./ws_pass) > $out/ws_pass.txt 2>&1; cat $out/ws_pass.txt

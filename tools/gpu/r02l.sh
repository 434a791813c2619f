out=gpurun_out/r02l; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3 or scaled_configs or row_split_virtual_ranks_full or cfg4_giant" > $out/pytest.log 2>&1; echo pytest=$?; tail -2 $out/pytest.log
timeout 900 python tools/a2_sweep.py cfg4 "TINV_A2=1" > $out/a2.txt 2>&1; echo a2=$?
cat $out/a2.txt

out=gpurun_out/r02n; mkdir -p $out
timeout 1800 python tools/mgs_vs_cwy.py --wide --full > $out/mgs_vs_cwy_wide.txt 2>&1; echo wide=$?
cat $out/mgs_vs_cwy_wide.txt

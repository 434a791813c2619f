for cfg in "1000 1000" "7 12" "5 10" "4 16" "3 8" "7 1000" "12 20"; do
  set -- $cfg
  r=$(TINV_RES_CS2=$1 TINV_RES_CS4=$2 timeout 120 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],3), d['info']['kernel_ms']['cwy'])")
  echo "cs2>=$1 cs4>=$2: $r"
done

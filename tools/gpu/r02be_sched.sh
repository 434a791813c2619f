for c in "cfg1" "cfg2" "type1 --n 2100" "type1 --n 4200" "type3 --n 2100" "type3 --n 4200"; do
  python tools/knob_sweep.py --config $c --knob TINV_CS_COST --sep ';' --values '1:1.5,2:1.25;1:1,2:1;1:2,2:1.5;1:1.25,2:1.1;1:1.5,2:1.25' --reps 20
  python tools/knob_sweep.py --config $c --knob TINV_SPLIT --sep ';' --values '2:1.15;2:1.0;2:1.3;2:1.15' --reps 20
done

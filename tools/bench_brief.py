import json, sys
for p in sys.argv[1:]:
    try:
        d = json.load(open(p))
    except Exception as exc:
        print(p, "unreadable", exc)
        continue
    i, r = d["info"], d["roofline"]
    print(f"{d['config']['name']}: {d['value']:.1f} eigvec/s  {d['ms_per_step']:.3f} ms/step  dom={r['kernel']} "
          f"{r['kernel_ms']:.3f} ms frac={r['frac']:.3f}  kernels={ {k: round(v, 3) for k, v in i['kernel_ms'].items()} }")
    print("   phases", {k: round(v, 3) for k, v in i["cwy_phase_ms"].items()}, "syncs", i["group_syncs"],
          "groups", i["ngroups"], "ctas", i["cwy_ctas"], "rc", i["return_codes"], "iters", i["iters_hist"])

import json, sys
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{f}: {d['value']:.2f} GF/s  {d['ms_per_step']:.3f} ms/step  e2e {d['e2e']['value']:.2f}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}  roof {r['kernel']} {r['bound']} frac {r['frac']:.3f}")
    for s, v in d["stages"].items():
        print(f"   {s:13s} {v['ms_per_launch']*1e3:9.1f} us  share {v['share']:.3f}  {v['GB_s']:7.0f} GB/s ({v['frac_hbm']:.2f})  {v['Gbfly_s']:6.0f} Gbfly/s ({v['frac_alu']:.2f})")
    for key in ("f1_cyclic", "f2_image", "f1_f2_cyclic_image", "f4_ts"):
        c = d.get(key)
        if c:
            print(f"   {key} (m={c['m']}): {c['value']:.2f} GF/s  {c['ms_per_step']:.3f} ms/step  "
                  f"ntts/transform {c.get('ntts_per_transform')}")

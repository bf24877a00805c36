import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    s = d["stage_ms"]
    print(f"{d['config']:10s} ep{d['ep']} n={d['tokens']:6d} eps={d['eps']:.2f} a={d['alpha']:.3f} "
          f"ms={d['ms_per_step']:.3f} tok/s={d['tokens_per_s']/1e6:.2f}M expTF={d['expert_tflops']:.0f} "
          f"up={s['expert_up']:.3f} dn={s['expert_down']:.3f} gate={s['gate']:.3f} srs={s['srs']:.3f} "
          f"disp={s['dispatch']:.3f} comb={s['combine_sag']:.3f} plan={s['plan']:.3f} route={s['route']:.3f}")

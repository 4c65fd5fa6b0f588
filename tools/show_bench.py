import json, sys
for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:
        print(path, 'ERR', e); continue
    print(f"== {d['config']['workload']}: {d['ms_per_step']:.3f} ms/iter; phases", {k: round(v, 3) for k, v in d['phases_ms'].items()})
    t = d['ttm_tree']
    print(f"   tree: {t['measured_ms']:.3f} ms vs roof {t['roofline_ms']:.3f} -> frac {t['roofline_frac']:.3f}, {t['tflops']:.2f} TF; P={t['p_fp64_tflops']:.2f}")
    print("   nodes:", " ".join(f"[{r['node']}:m{r['mode']} {r['bound'][0]} {r['ms']*1e3:.0f}us {r['frac']:.2f}]" for r in t['per_node']))
    if d.get('e2e'): print("   e2e", d['e2e']['value'])
    if d.get('cpu_baseline'): print("   cpu", d['cpu_baseline']['value'], d['cpu_baseline'].get('parity_first_iteration'))
    print("   fit", d['relative_fit'], "launches", d['gpu_launches'], "clocks", d['clocks'])

import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench_7b.json'))
for k in ('value', 'ms_per_step', 'pct_peak', 'tokens_per_s', 'layer_roofline_ms', 'layer_roofline_frac', 'gpu_launches', 'clocks'):
    print(k, d.get(k))
print('roofline', {k: d['roofline'][k] for k in ('kernel', 'bound', 'achieved', 'frac')})
for k, v in d['kernels'].items():
    print(f"{k:9s} {v['avg_ms']*1e3:8.1f}us {v['tflops']:7.1f}TF {v['gbs_paper']:7.0f}GB/s {v['bound']:6s} roof={v['roofline_ms']*1e3:6.1f}us frac={v['frac']:.2f}")

"""Summarise a bench.py JSON line (the last line of the given file)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value', 'ms_per_step', 'gpu_launches')})
print('latency', d.get('request_latency_us'))
print('roofline', d['roofline']['frac'], d['roofline']['achieved'], 'e2e', d.get('e2e', {}) and d['e2e']['value'])
cpu = d.get('cpu_baseline')
if cpu:
    print('cpu', cpu['value'], cpu['cores'], (cpu.get('single_thread') or {}).get('value'))
for n, l in (d.get('legs') or {}).items():
    if 'error' in l:
        print(n, l)
        continue
    if 'roofline' not in l:  # the TTFT-like consumer leg
        print(n, {k: v for k, v in l.items() if 'ms' in k or 'rel' in k or 'speed' in k})
        continue
    print(n, {k: l.get(k) for k in ('value', 'ms_per_step', 'hits_per_tier', 'build_seconds', 'request_latency_us')})
    print('    roof', l['roofline']['frac'], l['roofline']['achieved'], 'link', (l.get('link') or {}).get('frac'),
          (l.get('link') or {}).get('achieved_GBps'), 'overlapped', (l.get('overlapped_roofline') or {}).get('frac'),
          'hbm_budget', l.get('hbm_budget_bytes'))
ps = d.get('per_scheme')
if ps:
    print({k: (v['assemble_frac'], v['quantize_frac']) for k, v in ps.items()})

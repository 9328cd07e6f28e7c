import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
d = json.loads(l[-1])
print(round(d['value']), round(d['ms_per_step'], 1), round(d['pct_bf16_peak'], 4), 'e2e', (d.get("e2e") or {}).get("value"))
for k, v in d['kernels'].items():
    print(' ', k, {a: (round(b, 3) if isinstance(b, float) else b) for a, b in v.items() if a != 'note'})
tot = sum(v.get('ms_per_step', 0) for k, v in d['kernels'].items() if 'ms_per_step' in v and k not in ('bwd_dq', 'bwd_dkdv'))
print('  kernel sum ms/step', round(tot, 1), ' gap', round(d['ms_per_step'] - tot, 1))

import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
d = json.loads(l[-1])
print(round(d['value']), round(d['ms_per_step'], 1), round(d['pct_bf16_peak'], 4), 'e2e', (d.get("e2e") or {}).get("value"))
for k, v in d['kernels'].items():
    print(' ', k, {a: round(b, 3) for a, b in v.items()})
tot = sum(v.get('ms_per_step', 0) for k, v in d['kernels'].items() if 'ms_per_step' in v)
print('  kernel sum ms/step', round(tot, 1), ' gap', round(d['ms_per_step'] - tot, 1))

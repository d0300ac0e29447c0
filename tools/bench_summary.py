"""One-screen summary of a bench.py JSON line (value, per-e rooflines, configs)."""
import json,sys
d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith('{')][-1])
print('value',d['value'],'frac',d['roofline']['frac'],{k:(round(v['gnumbers_s'],1),round(v['imad_frac'],3)) for k,v in d['roofline']['per_exponent'].items()})
print('e2e',(d.get('e2e') or {}).get('value'),'clocks',d['clocks'])
for k,v in d.get('configs',{}).items():
  r=v.get('roofline') or {}
  print(k, round(v.get('value',0),2), v.get('unit'), r.get('frac'), r.get('kernel'), v.get('ms_per_step'))

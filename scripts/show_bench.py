import json, sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d = json.loads(line)
        r = d['roofline']
        print(f"ms/step {d['ms_per_step']:.2f}  cd {r['cd_ms_per_step']:.2f}  scan {r['scan_ms_per_step']:.2f} ({r['frac']:.3f} of {r['bound']} peak)  "
              f"ns/visit {r['cd_ns_per_visit']:.1f}  visits {r['cd_visits_per_step']:.0f}  phases/visit {json.dumps({k: round(v, 1) for k, v in r['cd_phase_cycles_per_visit'].items()})}  e2e {d['e2e']['value'] if d['e2e']['value'] is None else round(d['e2e']['value'], 4)}  path {d['path']}")

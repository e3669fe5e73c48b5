"""One-line summaries of bench JSON lines: python scripts/show_bench.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline", {})
    cpu = d.get("cpu_baseline", {}) or {}
    e2e = d.get("e2e", {}) or {}
    print(f"{d['config']['workload']:6s} {d['config'].get('resident','device'):6s} path {d['ms_per_step']:9.2f} ms | "
          f"roof {r.get('frac') or 0:.3f} ({r.get('achieved') or 0:.0f} {r.get('unit')}) scan {r.get('scan_ms_per_step') or 0:.1f} ms "
          f"cd {r.get('cd_ms_per_step') or 0:.1f} ms | e2e {e2e.get('value')} | cpu {cpu.get('value')} s x{cpu.get('lambdas')} lam "
          f"gpu_same {cpu.get('gpu_same_sample_s')} | launches {d.get('gpu_launches')} | clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")

import glob, json, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/perf_*.log")):
    try:
        l = json.loads([x for x in open(f) if x.startswith("{")][0])
    except Exception as e:
        print(f, "FAILED", open(f).read()[-300:]); continue
    r = l["roofline"]
    print(f"{f.split('/')[-1]:28s} path {l['value']*1e3:8.1f} ms  scan {r['scan_ms_per_step']:7.2f} ms @ {r['achieved']:7.0f} GB/s ({r['frac']*100:5.1f}%)  "
          f"cd {r['cd_ms_per_step']:8.2f} ms  visits {r.get('cd_visits_per_step',0):9.0f} ns/visit {r.get('cd_ns_per_visit',0):6.1f} kcyc/visit {r.get('cd_kernel_cycles_per_visit',0):6.1f} kernel-ms {r.get('cd_kernel_ms_per_step',0):7.2f}  e2e {l['e2e']['value']*1e3:7.1f} ms  phases {r.get('cd_phase_cycles_per_visit')}  launches {l['gpu_launches']}")

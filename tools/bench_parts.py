"""One line per bench log: step time and the per-kernel parts. python tools/bench_parts.py gpurun_out/v_*.log"""
import json
import sys

for f in sys.argv[1:]:
    try:
        j = json.loads([x for x in open(f) if x.startswith('{')][-1])
        k = j['kernels']
        p = k['enumerate'].get('parts_ms', {})
        print(f"{f.split('/')[-1]:22s} {j['ms_per_step']:8.3f} ms {j['value'] / 1e6:7.2f} M/s | yw {k['gemm_yw']['ms']:.3f} "
              f"sel {p.get('front', 0):.3f} states {p.get('states', 0):.3f} fb {p.get('fallback', 0):.3f} fin {p.get('finish', 0):.3f} "
              f"ytes {k['gemm_ytes']['ms']:.3f} final {k['finalize']['ms']:.3f} mstep {k['mstep']['ms']:.3f} "
              f"{j['clocks']['sm_mhz']} {j['clocks']['reasons']}")
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-300:])

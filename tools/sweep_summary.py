"""One line per workload from a gpu_sweep jsonl: ms/step, value, roofline frac, parity."""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    p = d.get("parity") or {}
    cfg = d.get("config", {})
    print(f"{cfg.get('workload', '?')[:28]:28s} {d['ms_per_step']:8.4f} ms  {d['value']:8.1f} {d['unit']:5s} "
          f"frac {r.get('frac', 0):.3f} ({r.get('bound')}) floor {r.get('floor_frac', 0):.3f}  "
          f"{r.get('kernel')}  parity {p.get('rel_fro', p.get('rel_l2_dist', 0)):.1e} "
          f"{p.get('sampled')}/{p.get('of')} {'PASS' if p.get('pass') else 'FAIL'}  "
          f"clk {d.get('clocks', {}).get('sm_mhz')}")

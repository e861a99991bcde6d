"""Print a one-line summary per bench JSON line found in the given files (skips non-JSON)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        lines = open(path).read().strip().splitlines()
    except OSError as e:
        print(path, "unreadable", e)
        continue
    got = False
    for ln in lines:
        try:
            d = json.loads(ln)
        except ValueError:
            continue
        if "value" not in d:
            print(path, d)
            continue
        got = True
        sp = d.get("stage_profile") or {}
        print(f"{path}: {d['config'].get('workload')} value {d['value']:.4g} {d['unit']} ms/step {d['ms_per_step']:.2f}"
              f" e2e {d.get('e2e', {}).get('value', float('nan')):.4g} prof_step {sp.get('step_ms') or float('nan'):.2f}"
              f" frac {d.get('roofline', {}).get('frac', float('nan')):.3f} launches {d.get('gpu_launches')}"
              f" clk {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
    if not got:
        print(path, "no bench line;", (lines[-1] if lines else "")[:200])

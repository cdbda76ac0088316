"""Print a one-line summary of bench.py JSON lines read from stdin (dev aid)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "roofline_run" not in d:
        print(line[:300])
        continue
    r, rr = d["roofline"], d["roofline_run"]
    print(f'{d["config"]["workload"][:5]} {d["ms_per_step"]:.3f} ms value={d["value"]:.3g} e2e={d["e2e"]["value"]:.3g} '
          f'tab={(d.get("e2e_table") or {}).get("value", 0):.3g} run_frac={rr["frac_of_roofline"]} '
          f'dom={r["kernel"]} {r["achieved"]}GB/s frac={r["frac"]} split={rr["kernel_split_ms"]}')

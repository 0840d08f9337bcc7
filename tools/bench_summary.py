"""Print the key fields of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline", {})
    print(f"{d['config']['workload'][:40]:40s} value={d['value']:.3f} {d['unit']} ms/step={d['ms_per_step']:.2f} "
          f"gemm={r.get('achieved', 0):.1f}TF step_frac={r.get('step_frac', 0):.3f} "
          f"e2e={d.get('e2e', {}).get('value', 0):.3f} clocks={d.get('clocks')}")

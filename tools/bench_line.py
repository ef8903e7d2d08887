"""Print the key fields of a bench.py JSON line read from stdin (diagnostics)."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
lines = [l for l in sys.stdin.read().strip().splitlines() if l.startswith("{")]
if not lines:
    print(tag, "no bench line")
    sys.exit(0)
d = json.loads(lines[-1])
rf = d.get("roofline", {})
print(tag, f"value={d.get('value'):.5f}", f"iters={d.get('config', {}).get('iterations')}",
      f"strip_us={rf.get('avg_launch_us', 0):.1f}", f"frac={rf.get('frac', 0):.3f}", f"kernel={rf.get('kernel')}",
      f"e2e={d.get('e2e', {}).get('value')}", f"clocks={d.get('clocks')}", flush=True)

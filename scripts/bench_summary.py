"""Print a one-line summary of bench.py's JSON line (stdin); extra argv words are prefixed."""
import json
import sys

lines = [ln for ln in sys.stdin.read().strip().splitlines() if ln.startswith("{")]
if not lines:
    print(" ".join(sys.argv[1:]), "NO JSON LINE")
    sys.exit(0)
x = json.loads(lines[-1])
p, s = x.get("phases_ms", {}), x.get("stats", {})
rf = x.get("roofline") or {}
print(" ".join(sys.argv[1:]), f"value {x['value']:.4g} ms/step {x['ms_per_step']:.3f} bis {p.get('root_bisection', 0):.3f} "
      f"clu {p.get('clusters', 0):.3f} rqi {p.get('singletons', 0):.3f} root {p.get('split_root', 0):.3f} "
      f"rounds {s.get('rounds')} negx {s.get('negcount_x')} iters {s.get('rqi_iters')} fb {s.get('rqi_fallbacks')} "
      f"ho {s.get('rqi_handover')}/{s.get('ho_twist')}/{s.get('ho_fixed')}/{s.get('ho_rqc')} wide {s.get('seg_wide')} "
      f"roof {rf.get('kernel', '')[:12]} frac {rf.get('frac', 0):.3f}", flush=True)

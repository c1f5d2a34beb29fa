"""Print the headline numbers and per-layer ms of a bench.py log."""
import json
import sys

for f in sys.argv[1:]:
    for ln in open(f):
        if ln.startswith("{"):
            d = json.loads(ln)
            r = d.get("roofline", {})
            print(f, "value %.0f e2e %.0f frac %.3f" % (d["value"], d["e2e"]["value"], r.get("frac") or 0), d.get("op_ms"))
            for k, v in (r.get("per_layer_ms") or {}).items():
                print("   %-30s %.4f" % (k, v))

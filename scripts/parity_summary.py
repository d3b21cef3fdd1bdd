"""Summarise UA_PARITY_LOG JSON lines (tests/parity.py) into
profiles/r02_parity_margins.json: per gate kind, the worst elementwise margin
(err / bound), the worst Gate-A fraction and the worst relative L2.
    python scripts/parity_summary.py gpurun_out/parity_*.jsonl"""
import collections
import json
import os
import sys

rows = []
for f in sys.argv[1:]:
    rows += [json.loads(line) for line in open(f)]
summ = collections.defaultdict(lambda: dict(n=0, worst_elt=0.0, worst_elt_test=None, worst_gate_a=0.0,
                                            worst_rel_l2=0.0, worst_q7=0.0, q7_fail=0))
for r in rows:
    s = summ[r["gate"]]
    s["n"] += 1
    if (r.get("elt_margin") or 0) > s["worst_elt"]:
        s["worst_elt"], s["worst_elt_test"] = r["elt_margin"], r["test"]
    if r.get("gate_a_max_frac") is not None:
        s["worst_gate_a"] = max(s["worst_gate_a"], r["gate_a_max_frac"])
    if r.get("rel_l2") is not None:
        s["worst_rel_l2"] = max(s["worst_rel_l2"], r["rel_l2"])
    if r.get("q7_margin") is not None:
        s["worst_q7"] = max(s["worst_q7"], r["q7_margin"])
        s["q7_fail"] += r["q7_margin"] > 1.0
out = {"_about": "Achieved margins of the parity gates (tests/parity.py with UA_PARITY_LOG) over the GPU suites in "
                 + ", ".join(os.path.basename(f) for f in sys.argv[1:]) + ".  worst_elt = max over elements of "
                 "err / elementwise bound (passes <= 1); worst_gate_a = max-abs / north-star bound (1e-2 out, 2e-2 "
                 "grads, 1e-3 lse; N(0,1) cases); worst_rel_l2 against the 1e-2 gate; worst_q7 / q7_fail = the same error "
                 "against SURVEY Q7's original elementwise bound 1e-3 + 2^-6 |ref| (not enforced, DESIGN R7).",
       "calls": len(rows), "gates": summ}
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/r02_parity_margins.json", "w"), indent=1)
print(json.dumps(out, indent=1))

"""Summarise an ncu --page source --csv dump: top instructions by stall samples with
their dominant stall reasons.  usage: python tools/ncu_hot.py <csv> [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
I = {h: i for i, h in enumerate(hdr)}
seen, data = set(), []
for r in rows[2:]:
    if len(r) != len(hdr) or r[I["Address"]] in seen:
        continue
    seen.add(r[I["Address"]])
    data.append(r)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def g(r, k):
    try:
        return float(r[I[k]] or 0)
    except ValueError:
        return 0.0


tot = sum(g(r, "Warp Stall Sampling (All Samples)") for r in data)
agg = {c: sum(g(r, c) for r in data) for c in stall_cols}
print("total samples", tot)
print("by reason:", ", ".join(f"{c[6:]}={v / tot:.1%}" for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
for idx, r in sorted(enumerate(data), key=lambda ir: -g(ir[1], "Warp Stall Sampling (All Samples)"))[:n]:
    reasons = sorted(((c[6:], g(r, c)) for c in stall_cols), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{k}:{int(v)}" for k, v in reasons if v > 0)
    print(f"{idx:5d} {r[I['Source']].strip()[:58]:58s} {int(g(r, 'Warp Stall Sampling (All Samples)')):5d} ex={int(g(r, 'Instructions Executed')):8d} {rs}")

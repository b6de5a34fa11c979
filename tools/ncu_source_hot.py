"""Summarise an `ncu --page source --csv --print-source sass` export: per-instruction stall samples
for the first kernel in the file, top-N instructions and the stall mix by opcode."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    name = rows[0][1] if len(rows[0]) > 1 else "?"
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    body = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            break  # next kernel
        body.append(r)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    byop = collections.defaultdict(collections.Counter)
    for r in body:
        op = r[idx["Source"]].strip().split()[0] if r[idx["Source"]].strip() else "?"
        if op.startswith("@"):
            op = r[idx["Source"]].strip().split()[1]
        for s in stalls:
            v = int(r[idx[s]] or 0)
            tot[s] += v
            byop[op.split(".")[0]][s] += v
    print(name[:120])
    T = sum(tot.values())
    print("total samples", T)
    for s, v in tot.most_common():
        if v:
            print(f"  {s:24s} {v:8d} {100*v/T:5.1f}%")
    print("by opcode (samples, top stalls):")
    ops = sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))
    for op, c in ops[:15]:
        n = sum(c.values())
        print(f"  {op:10s} {n:8d} {100*n/T:5.1f}%  " + ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(4) if v))
    print("hot instructions:")
    hot = sorted(body, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[:top]
    for r in hot:
        c = {s: int(r[idx[s]] or 0) for s in stalls}
        top3 = sorted(c.items(), key=lambda kv: -kv[1])[:3]
        print(f"  {r[idx['Address']][-5:]} {r[idx['Warp Stall Sampling (All Samples)']]:>6s} {r[idx['Source']].strip()[:60]:60s} "
              + " ".join(f"{k[6:]}={v}" for k, v in top3 if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

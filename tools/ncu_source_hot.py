"""Summarise an `ncu --page source --csv --print-source sass` export: per-instruction stall samples
for the K-th kernel in the file (default the first; `all` = every kernel, stall mix only), top-N
instructions and the stall mix by opcode.

    python tools/ncu_source_hot.py file.csv [top] [kernel index | all]"""
import collections
import csv
import sys


def split_kernels(rows):
    """[(name, header, body rows)]: a kernel section starts with a short name row followed by the header."""
    out, i = [], 0
    while i < len(rows):
        if i + 1 < len(rows) and "Source" in rows[i + 1] and "Source" not in rows[i]:
            name = rows[i][1] if len(rows[i]) > 1 else "?"
            hdr = rows[i + 1]
            j = i + 2
            body = []
            while j < len(rows) and len(rows[j]) == len(hdr) and "Source" not in rows[j]:
                body.append(rows[j])
                j += 1
            out.append((name, hdr, body))
            i = j
        else:
            i += 1
    return out


def main(path, top=40, which=0):
    ks = split_kernels(list(csv.reader(open(path))))
    if which == "all":
        for k in range(len(ks)):
            report(*ks[k], top=0)
        return
    report(*ks[int(which)], top=top)


def report(name, hdr, body, top=40):
    idx = {h: i for i, h in enumerate(hdr)}
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
    if not top:
        return
    print("hot instructions:")
    hot = sorted(body, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[:top]
    for r in hot:
        c = {s: int(r[idx[s]] or 0) for s in stalls}
        top3 = sorted(c.items(), key=lambda kv: -kv[1])[:3]
        print(f"  {r[idx['Address']][-5:]} {r[idx['Warp Stall Sampling (All Samples)']]:>6s} {r[idx['Source']].strip()[:60]:60s} "
              + " ".join(f"{k[6:]}={v}" for k, v in top3 if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, sys.argv[3] if len(sys.argv) > 3 else 0)

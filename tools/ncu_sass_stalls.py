"""Aggregate ncu per-SASS-instruction warp-stall samples by opcode and by code region.

    python tools/ncu_sass_stalls.py gpurun_out/ncu/bert512_sass.csv [--top 25]

Input: `ncu -i REP --page source --csv --print-source sass`.  Prints the samples per
opcode (with the dominant stall reasons) and the hottest instructions in address order.
"""
import argparse
import csv
import collections
import io


def load(path):
    txt = open(path).read()
    i = txt.index('"Kernel Name"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    rows = rows[1:]  # the first row is the kernel-name header
    hdr = rows[0]
    out = []
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        out.append(dict(zip(hdr, r)))
    return hdr, out


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    hdr, rows = load(a.csv)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    total = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rows)
    by_op = collections.defaultdict(lambda: collections.Counter())
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        c = by_op[op.split(".")[0]]
        c["samples"] += num(r["Warp Stall Sampling (All Samples)"])
        for s in stalls:
            c[s] += num(r[s])
    print(f"total samples {total:.0f}")
    for op, c in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[: a.top]:
        top = sorted(((k, v) for k, v in c.items() if k != "samples"), key=lambda kv: -kv[1])[:4]
        print(f"{op:22s} {100 * c['samples'] / total:5.1f}%  " + "  ".join(f"{k[6:]}={100 * v / total:.1f}" for k, v in top))
    print("\nhottest instructions:")
    hot = sorted(rows, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[: a.top]
    for r in sorted(hot, key=lambda r: int(r["Address"], 16)):
        s = num(r["Warp Stall Sampling (All Samples)"])
        top = sorted(((k, num(r[k])) for k in stalls), key=lambda kv: -kv[1])[:2]
        print(f"{r['Address']} {100 * s / total:5.2f}% {r['Source'][:60]:60s} " + " ".join(f"{k[6:]}={v:.0f}" for k, v in top))


if __name__ == "__main__":
    main()

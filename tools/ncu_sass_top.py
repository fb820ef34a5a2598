"""Per-kernel SASS hot spots from an ncu report's source page (--page source --csv
--print-source sass): top instructions by warp-stall samples with their dominant
stall reasons, and executed-instruction totals.
Usage: ncu -i rep --page source --csv --print-source sass > s.csv; python tools/ncu_sass_top.py s.csv [top]"""
import csv
import sys


def sections(path):
    cur = None
    for r in csv.reader(open(path)):
        if r and r[0] == "Kernel Name":
            if cur:
                yield cur
            cur = {"name": r[1], "hdr": None, "rows": []}
        elif cur is not None and cur["hdr"] is None:
            cur["hdr"] = r
        elif cur is not None:
            cur["rows"].append(r)
    if cur:
        yield cur


def main():
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    for sec in sections(sys.argv[1]):
        h = {k: i for i, k in enumerate(sec["hdr"])}
        rows = [r for r in sec["rows"] if len(r) == len(sec["hdr"])]
        f = lambda r, k: float(r[h[k]] or 0) if k in h else 0.0
        tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in rows)
        inst = sum(f(r, "Instructions Executed") for r in rows)
        stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
        agg = {k: sum(f(r, k) for r in rows) for k in stalls}
        print(f"== {sec['name'][:100]}\n   samples {tot:.0f}  warp-instructions executed {inst:.0f}")
        print("   stalls: " + ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.0f}%" for k, v in
                                        sorted(agg.items(), key=lambda kv: -kv[1])[:6]))
        for r in sorted(rows, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
            rs = sorted(((f(r, k), k[6:]) for k in stalls), reverse=True)[:2]
            print(f"   {f(r, 'Warp Stall Sampling (All Samples)'):6.0f} {r[h['Address']]:>6} {r[h['Source']][:60]:60s} "
                  + " ".join(f"{n}={v:.0f}" for v, n in rs))


if __name__ == "__main__":
    main()

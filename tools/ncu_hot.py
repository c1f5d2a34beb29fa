"""Hot SASS lines of an ncu --page source --csv export: stall samples and executed counts.
    python tools/ncu_hot.py source.csv [top]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:]]
    S = lambda d: int(d.get("Warp Stall Sampling (All Samples)") or 0)
    N = lambda d: int(d.get("Warp Stall Sampling (Not-issued Samples)") or 0)
    E = lambda d: int(d.get("Instructions Executed") or 0)
    tot_s, tot_e = sum(map(S, data)), sum(map(E, data))
    print(f"samples {tot_s}  warp-instructions {tot_e}")
    hot = sorted(range(len(data)), key=lambda i: S(data[i]), reverse=True)[:top]
    for i in sorted(hot):
        d = data[i]
        print(f"{i:6d} {E(d):10d} {S(d):6d} {N(d):6d}  {d['Source'][:110]}")


if __name__ == "__main__":
    main()

"""Per-source-line stall-reason breakdown from an ncu report (warp-state sampling).

    python scripts/ncu_stalls.py report.ncu-rep [n_lines] [line_lo line_hi]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    path, hdr, lines = None, None, []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r or not r[0].isdigit():
            continue
        ln = int(r[0])
        rec = dict(zip(hdr, r))
        try:
            tot = int(rec.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if tot == 0 or not (lo <= ln <= hi):
            continue
        st = {k[6:]: int(v) for k, v in rec.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
        lines.append((tot, f"{path}:{ln}", r[1].strip()[:60], st))
    total = sum(l[0] for l in lines) or 1
    for tot, loc, src, st in sorted(lines, key=lambda x: (x[0], x[1]), reverse=True)[:n]:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
        print(f"{tot / total:6.1%} {loc:22s} {src:60s} " + " ".join(f"{k}={v}" for k, v in top))


if __name__ == "__main__":
    main()

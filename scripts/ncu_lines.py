"""Top CUDA source lines of an ncu report by warp-stall samples and executed instructions.

    python scripts/ncu_lines.py report.ncu-rep [n]
"""
import csv
import io
import subprocess
import sys


def main(rep, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    path, lines = None, []
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] not in ("", "Function Name"):
            try:
                samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
                inst = int(r[hdr.index("Instructions Executed")])
            except (ValueError, IndexError):
                continue
            lines.append((samp, inst, f"{path}:{r[0]}", r[1].strip()[:90]))
    tot_s = sum(l[0] for l in lines) or 1
    tot_i = sum(l[1] for l in lines) or 1
    print(f"total samples {tot_s}  instructions {tot_i}")
    for s, i, loc, src in sorted(lines, reverse=True)[:n]:
        print(f"{s/tot_s:6.1%} {i/tot_i:6.1%}  {loc:22s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

"""Warp-stall samples per CUDA source line from an ncu report (--import-source on,
compiled with -lineinfo).  Inlined helpers are attributed to their own lines.

python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kernel=None, top=30):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ex = hdr.index("Instructions Executed")
    lines = []
    for r in rows:
        if len(r) > si and r[0] not in ("", "Line No") and r[si] not in ("-", ""):
            try:  # source lines with embedded quotes can shift columns: skip them
                lines.append((int(r[0]), float(r[si]), r[ex], r[1].strip()))
            except ValueError:
                continue
    tot = sum(v for _, v, _, _ in lines) or 1.0
    print(f"total samples {tot:.0f}")
    for ln, v, e, src in sorted(lines, key=lambda t: -t[1])[:int(top)]:
        print(f"{ln:5d} {100 * v / tot:5.1f}%  {e:>10s}  {src[:100]}")


if __name__ == "__main__":
    main(*sys.argv[1:])

"""Summarise `nvcc -Xptxas -v` output: registers and spills per kernel."""
import re
import subprocess
import sys


def main(src, pattern=""):
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
           "-std=c++17", "-Xptxas", "-v", "-I", "include", "-I", "paper_2110_08450_b200/csrc",
           "-c", src, "-o", "/tmp/_ptxas.o"]
    out = subprocess.run(cmd, capture_output=True, text=True).stderr
    name = None
    spill = None
    for line in out.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            spill = int(m.group(1))
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and name and pattern in name:
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            print(f"{int(m.group(1)):4d} regs {spill:5d} spill  {dem[:150]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")

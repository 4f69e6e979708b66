"""Per-kernel register / spill report of the product build (ptxas -v).

    python scripts/ptxas_spills.py [--all]
Prints one line per dls_search_kernel instantiation (N, VS, EMIT, CLOSE, LOOK):
registers, stack frame, spill stores / loads.  Without --all only kernels with a
non-zero spill are listed.
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1709_02599_b200", "csrc", "count.cu")


def main():
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
           "-Xptxas=-v", "-c", "-diag-suppress", "177", "-I", os.path.join(ROOT, "include"),
           "-o", "/tmp/_spills.o", SRC] + [a for a in sys.argv[1:] if a.startswith("-D")]
    out = subprocess.run(cmd, capture_output=True, text=True).stderr
    cur = None
    rows = []
    for line in out.splitlines():
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            rows.append([cur, *map(int, m.groups()), None])
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and rows and rows[-1][4] is None:
            rows[-1][4] = int(m.group(1))
    for name, frame, st, ld, regs in rows:
        k = re.search(r"dls_search_kernel<([^>]*)>", name)
        if not k:
            continue
        if st or ld or "--all" in sys.argv:
            print("%-40s regs %3s  frame %3d  spill st %3d ld %3d" % (k.group(1), regs, frame, st, ld))


if __name__ == "__main__":
    main()

"""Stall-reason and pipe summary of one ncu --set full report (raw page):
    python scripts/ncu_stalls.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = {h: v for h, v in zip(rows[0], rows[2])}

    def num(k):
        return float(d[k].replace(",", ""))

    keys = [k for k in d if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k]
    tot = sum(num(k) for k in keys)
    print("| stall reason (warp samples) | share |\n|---|---|")
    for k in sorted(keys, key=lambda k: -num(k)):
        if num(k) / tot > 0.01:
            print("| %s | %.1f%% |" % (k.replace("smsp__pcsamp_warps_issue_stalled_", ""), 100 * num(k) / tot))
    print()
    print("| unit | busy |\n|---|---|")
    for k, name in (("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots"),
                    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe"),
                    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe"),
                    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe (instructions)"),
                    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory data pipe (wavefronts)"),
                    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps per scheduler cycle (of 8)")):
        if k in d:
            print("| %s | %s |" % (name, d[k]))


if __name__ == "__main__":
    main()

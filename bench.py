#!/usr/bin/env python
"""Benchmark: exhaustive enumeration of order-8 diagonal Latin squares, first row
fixed (BASELINE.json config 3; 7 447 587 840 squares), on B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one pass of the hot path over the whole workload: every one of the
547 896 depth-14 workunits (first row + both diagonals, P:481 / Fig. 1 order)
searched by the sm_100a kernel down to the two-row level (the last two open
rows are counted in closed form).

value  : squares/s with the workunits resident in HBM; per-step CUDA events on
         the launch stream, L2 flushed (256 MiB write) before every step, max
         over ranks.
e2e    : the same through the public API with HOST buffers each step:
         dls_split on the host -> dls_count(host records) -> H2D copy, search,
         D2H of the count, all inside the timed region.
N > 1  : torchrun, one process per GPU; the workunits are dealt round-robin to
         ranks (no data-path collective), one int64 all_reduce of the count at the
         end of each step; total work is fixed ("scaling": "strong").
--impl reference : the CPU oracle (oracle/, the only reference this paper-only
         task has) on bounded samples of the same workunits, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_ORDER = 8
SYMMETRIC = False
WORKLOAD = "dls8_first_row_fixed_full"
METRIC = "diagonal Latin squares enumerated/sec"
UNIT = "squares/s"
NCU_JSON = "r2_ncu_close.json"  # the committed ncu --set full capture of the timed kernel
                                 # (used only if its count_cu_sha matches the source)
# Algorithmic integer operations per search node: one pass
# of Alg. 4's loop body for a non-diagonal cell:
#   CR = Rows|Columns (1), L = AllN^CR (1), L != 0 test (1), b = L&-L (2),
#   mark Rows/Columns (2), unmark Rows/Columns (2), L &= L-1 (2), loop exit test
#   amortised (1)  -> 12
OPS_PER_NODE = 12
# Algorithmic integer operations per two-row closure,
# |J| = 6 open columns for the N=8 plan: per column complement (1), isolate the
# low value (2), fold it into t (1) -> 24; GF(2) elimination: per pivot isolate
# (2) + rank (1) + t update (2) -> 30, per pair of columns test + xor (2) x 15 ->
# 30; final test and shift (3) -> 87
OPS_PER_CLOSURE = 87
DLS8_COUNT = 7447587840
# nodes of the full Alg. 4 tree below the 547 896 workunits (every one of the 42
# cells assigned one by one, as the paper's loop nest does): the plain search
# (DLS_CLOSE=0) reports it, profiles/r2_ab_step.log; node parity with the oracle
# on sampled workunits: tests/test_gpu_parity.py
DLS8_ALG4_TREE_NODES = 368133443872
PAPER_CONTEXT = "paper: 5.8e6 DLS8 squares/s on one core of an Intel Core i7-6770 (Table 1, P:281); context only"


def peaks():
    p = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except OSError:
        pass
    return p


def int_issue_peak_tops(sm_mhz: float, sms: int = 148) -> float:
    """Integer-issue roofline: 148 SMs x 4 SMSPs x 1 warp-instruction/clk
    x 32 lanes at the SM clock, in tera integer-lane-ops/s."""
    return sms * 4 * 32 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = "/tmp/dls_clocks_%d_%d.csv" % (os.getpid(), gpu_index)

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx.append(float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_workunits():
    """The workunits of the config from the ORACLE alone (its plan and prefix
    enumeration): every consistent assignment of the first `depth` plan
    cells, depth = the first prefix length covering both diagonals (Fig. 1)."""
    import oracle
    plan = oracle.plan(N_ORDER)
    diag = {i * N_ORDER + j for i in range(1, N_ORDER) for j in (i, N_ORDER - 1 - i)}
    depth = next(k for k in range(len(plan) + 1) if diag <= set(plan[:k]))
    recs = oracle.prefixes(N_ORDER, SYMMETRIC, oracle.first_row_grid(N_ORDER), plan, depth)
    return plan, depth, recs


def run_reference(args):
    """--impl reference: the CPU oracle on bounded samples of the workunits
    (loads only oracle/; no product code)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    plan, depth, recs = oracle_workunits()
    order = plan[depth:]
    rng = np.random.default_rng(20260)
    budget = float(os.environ.get("DLS_REF_STEP_SECONDS", "4"))
    times, squares, nodes, done = [], 0, 0, 0
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        s_sq = s_nd = 0
        while time.perf_counter() - t0 < budget:
            r = recs[int(rng.integers(len(recs)))]
            c, nd = oracle.count(N_ORDER, SYMMETRIC, r, order)
            s_sq += c
            s_nd += nd
            if step >= args.warmup:
                done += 1
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            squares += s_sq
            nodes += s_nd
    total_t = sum(times)
    v = squares / total_t if total_t else 0.0
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / max(args.steps, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": WORKLOAD, "n": N_ORDER, "prefix_depth": depth,
                                            "sample": "random workunits, %.0f s of oracle time per step" % budget},
            "nodes_per_sec": nodes / total_t if total_t else 0.0,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": "%d random depth-%d workunits of %d (N=8, row 0 fixed), %.0f s/step"
                                       % (done, depth, len(recs), budget)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "context": PAPER_CONTEXT}
    print(json.dumps(line), flush=True)


def pick_depth(world: int, lanes_per_gpu: int = 148 * 1024) -> int:
    """Smallest split depth >= the diagonal depth giving every rank at least ~3.5
    workunits per lane (the warp-level donation absorbs the remaining tail)."""
    from paper_1709_02599_b200 import _binding as B
    d = B.dls_plan(N_ORDER, SYMMETRIC)[2]
    lib = B.load()
    while lib.dls_split(N_ORDER, int(SYMMETRIC), 1, d, None, 0) < 3.5 * lanes_per_gpu * world:
        d += 1
    return d


def cpu_baseline(seconds: float):
    """The oracle, as it stands, on random workunits it enumerates itself."""
    import oracle
    plan, depth, recs = oracle_workunits()
    order = plan[depth:]
    rng = np.random.default_rng(1709)
    t0 = time.perf_counter()
    sq = nd = k = 0
    while time.perf_counter() - t0 < seconds:
        r = recs[int(rng.integers(len(recs)))]
        c, n_ = oracle.count(N_ORDER, SYMMETRIC, r, order)
        sq += c
        nd += n_
        k += 1
    dt = time.perf_counter() - t0
    return {"value": sq / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": "%d random depth-%d workunits of N=8 (row 0 fixed), %.1f s single-thread; "
                      "nodes/s %.3g" % (k, depth, dt, nd / dt)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_1709_02599_b200 as D
    from paper_1709_02599_b200 import _binding as B

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()

    from paper_1709_02599_b200.dist import allreduce_count, allreduce_max, shard_workunits
    depth = pick_depth(world)
    recs_all = D.dls_split(N_ORDER, depth, SYMMETRIC)
    mine = shard_workunits(recs_all, rank, world)    # round-robin shard of the workunits
    d_recs = torch.from_numpy(mine).to(dev)
    d_stats = torch.zeros(B.DLS_STATS_WORDS, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    def reduce_count(x):
        return allreduce_count(x, device=dev)

    def device_step():
        B.dls_count_async(N_ORDER, depth, d_recs, None, d_stats, SYMMETRIC, stream=stream.cuda_stream)

    # ---- warm-up
    for _ in range(args.warmup):
        device_step()
    torch.cuda.synchronize()

    # ---- timed: K steps, per-step events on the launch stream, L2 flushed in between
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    counts, nodes_l, events_l = [], [], []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            device_step()
            evs[i][1].record(stream)
            st = d_stats.cpu()
            counts.append(reduce_count(int(st[0])))
            nodes_l.append(reduce_count(int(st[1])))
            events_l.append(reduce_count(int(st[8])))
            assert int(st[2]) == 0
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    local_ms = sum(step_ms)
    total_ms = allreduce_max(local_ms, device=dev)
    clocks = clk.summary()
    squares = counts[0]
    # every timed step must reproduce P:476 and visit the same tree
    if any(c != DLS8_COUNT for c in counts) or len(set(nodes_l)) != 1 or len(set(events_l)) != 1:
        raise SystemExit("timed steps disagree: counts %s nodes %s closures %s" % (counts, nodes_l, events_l))
    value = squares * args.steps / (total_ms / 1e3)
    nodes_per_sec = nodes_l[0] * args.steps / (total_ms / 1e3)

    # ---- e2e: public API with host buffers, split + H2D + search + D2H inside.
    # The records are written into pinned host memory (allocated once, like any
    # serving buffer); each step re-runs the host split into it, then dls_count
    # copies them to HBM, searches and returns the count.
    e2e = None
    if not args.no_e2e:
        lib = B.load()
        n_all = int(recs_all.shape[0])
        pin_all = torch.empty((n_all, N_ORDER, N_ORDER), dtype=torch.uint8).pin_memory()
        pin_mine = pin_all if world == 1 else torch.empty((len(mine), N_ORDER, N_ORDER), dtype=torch.uint8).pin_memory()

        def e2e_step():
            got = lib.dls_split(N_ORDER, int(SYMMETRIC), 1, depth, pin_all.data_ptr(), n_all)
            assert got == n_all
            if world > 1:
                pin_mine.numpy()[:] = pin_all.numpy()[rank::world]
            tot, _ = D.dls_count(N_ORDER, depth, pin_mine, SYMMETRIC, stream=stream.cuda_stream)
            return reduce_count(tot)

        e2e_step()                                   # warm-up
        e2e_steps = max(1, min(args.steps, 3))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            assert e2e_step() == DLS8_COUNT
        torch.cuda.synchronize()
        el = allreduce_max(time.perf_counter() - t0, device=dev)
        e2e = {"value": DLS8_COUNT * e2e_steps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(pin_mine.numel()), "d2h_bytes_per_step": 8 * B.DLS_STATS_WORDS,
               "includes": "host dls_split into pinned memory + H2D of the workunits + search + D2H of the count"}

    if rank == 0:
        pk = peaks()
        sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
        peak = int_issue_peak_tops(sm_mhz)
        per_launch_ms = local_ms / args.steps
        ops = nodes_l[0] * OPS_PER_NODE + events_l[0] * OPS_PER_CLOSURE
        achieved = ops / world / (per_launch_ms / 1e3) / 1e12
        ncu, ncu_note = {}, ""
        try:
            import hashlib
            with open(os.path.join(ROOT, "profiles", NCU_JSON)) as f:
                ncu = json.load(f)
            src = os.path.join(ROOT, "paper_1709_02599_b200", "csrc", "count.cu")
            sha = hashlib.sha256(open(src, "rb").read()).hexdigest()[:16]
            if ncu.get("count_cu_sha") != sha:
                ncu_note = "capture %s is of another count.cu (%s != %s): ncu fields omitted" % (
                    NCU_JSON, ncu.get("count_cu_sha"), sha)
                ncu = {}
        except (OSError, ValueError):
            ncu, ncu_note = {}, "no capture %s" % NCU_JSON
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": N_ORDER, "symmetric": SYMMETRIC, "first_row_fixed": True,
                       "prefix_depth": depth, "n_prefix": int(recs_all.shape[0]),
                       "squares_per_step": squares, "nodes_per_step": nodes_l[0],
                       "closures_per_step": events_l[0], "search_levels": B.dls_search_levels(N_ORDER, depth),
                       "l2": "flushed before every step (256 MiB device write)",
                       "parallelism": "workunits round-robin over %d rank(s)" % world},
            "nodes_per_sec": nodes_per_sec,
            "closures_per_sec": events_l[0] * args.steps / (total_ms / 1e3),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                         "frac": achieved / peak,
                         "traffic": (ncu["dram_read_bytes"] + ncu["dram_write_bytes"]) if ncu else None,
                         "traffic_note": ncu_note or ("DRAM bytes per launch from the committed ncu --set full "
                                                      "capture (profiles/%s) = the 35 MB of workunit records: "
                                                      "the search itself never touches HBM" % NCU_JSON),
                         "ops_per_node": OPS_PER_NODE, "ops_per_closure": OPS_PER_CLOSURE,
                         # context: the same time against the work of the paper's own loop
                         # nest (its full tree, 12 ops per node) -- what the closure saves
                         # shows up here, not in frac
                         "frac_of_peak_alg4_full_tree": (DLS8_ALG4_TREE_NODES * OPS_PER_NODE / world
                                                         / (per_launch_ms / 1e3) / 1e12) / peak,
                         "alu_pipe_busy_ncu": (ncu.get("alu_pipe_pct", 0) / 100.0) if ncu else None,
                         "fmaheavy_pipe_busy_ncu": (ncu.get("fmaheavy_pipe_pct", 0) / 100.0) if ncu else None,
                         "issue_slots_busy_ncu": (ncu.get("issue_slots_busy_pct", 0) / 100.0) if ncu else None,
                         # issue slots, ALU pipe, FMA-heavy pipe and the shared-memory
                         # data pipe are all 70-90% busy
                         "smem_pipe_busy_ncu": (ncu.get("smem_lsu_wavefronts_pct", 0) / 100.0) if ncu else None,
                         "note": "integer-issue roofline at %.0f MHz (MEASURED_PEAKS sm_max_mhz): 148 SMs x 4 SMSP x "
                                 "32 lanes; achieved = (%d int ops x nodes the kernel visits (Alg. 4 loop body) + "
                                 "%d x two-row closures) / kernel time" % (sm_mhz, OPS_PER_NODE, OPS_PER_CLOSURE)},
            "clocks": clocks,
            "gpu_launches": args.steps * B.dls_kernel_launches(),
            "wall_ms_timed_region": t_wall * 1e3,
            "context": PAPER_CONTEXT,
        }
        if e2e:
            line["e2e"] = e2e
        if world == 1 and args.cpu_seconds > 0:
            line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

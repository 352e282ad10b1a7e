#!/usr/bin/env python
"""bench.py — edges coloured per second (GTEPS) of the B200 SGR colouring path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat24] [--impl ours|reference]

A "step" is one whole gc_color call (ingest + every SGR round + finalize) on the
BASELINE.json workload, inputs resident in HBM.  Prints ONE JSON line (rank 0).
See DESIGN.md §7 for the roofline bytes, the CPU baseline sample and the e2e leg.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges colored/sec (GTEPS)"
UNIT = "GTEPS"

# bounded CPU-oracle samples of each workload family (~10-30 s of single-core CPU work)
CPU_SAMPLES = {
    "rmat24": ("rmat", dict(scale=22, edge_factor=16)),
    "rmat16": ("rmat", dict(scale=16, edge_factor=8)),
    "stencil128": ("stencil", dict(nx=96)),
    "mesh8192": ("mesh", dict(rows=4096, cols=4096, p_delete=0.3)),
    "rmat27": ("rmat", dict(scale=21, edge_factor=16)),
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def sample_graph(cfg):
    import workloads as wl
    kind, kw = CPU_SAMPLES[cfg]
    if kind == "rmat":
        return wl.rmat(kw["scale"], kw["edge_factor"]), f"R-MAT scale {kw['scale']} ef {kw['edge_factor']} (same generator/params as {cfg})"
    if kind == "stencil":
        return wl.stencil27(kw["nx"]), f"27-point stencil {kw['nx']}^3 (same generator as {cfg})"
    return wl.mesh2d(kw["rows"], kw["cols"], kw["p_delete"]), f"mesh {kw['rows']}x{kw['cols']} 30% deleted (same generator as {cfg})"


def cpu_oracle_gteps(cfg):
    """Time the CPU oracle as it stands (single-threaded C) on a bounded sample."""
    import oracle
    g, desc = sample_graph(cfg)
    t0 = time.perf_counter()
    _, nc, r = oracle.sgr(g)
    dt = time.perf_counter() - t0
    return dict(value=g.m / dt / 1e9, unit=UNIT, cores=1, kind="oracle",
                sample=f"{desc}: n={g.n} m={g.m}, full oracle_sgr run, {dt:.2f} s, {r} rounds, {nc} colors",
                seconds=dt)


_REASONS = {
    "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
    "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
    "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
}


def _clock_proc(index, conn):
    """Sampler process body: SM clock + throttle reasons every 5 ms until told to stop."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        conn.send("no nvml")
        return
    samples, reasons = [], set()
    conn.send("ready")
    while not conn.poll():
        try:
            samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            reasons.update(k for k, bit in _REASONS.items() if r & bit and k != "gpu_idle")
        except Exception:
            pass
        time.sleep(0.005)
    conn.send((samples, sorted(reasons), max_mhz))


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs, in a
    separate process (a sampling thread here would compete for the GIL with the timed loop's
    host side: measured up to +0.7 ms per step on the mesh)."""

    def __init__(self, index):
        self.index = index
        self._p = None
        self._c = None

    def start(self):
        if os.environ.get("GC_BENCH_CLOCKS") == "0":  # diagnostics only: no sampling
            return self
        try:
            import multiprocessing as mp
            ctx = mp.get_context("spawn")
            self._c, child = ctx.Pipe()
            self._p = ctx.Process(target=_clock_proc, args=(self.index, child), daemon=True)
            self._p.start()
            if not self._c.poll(60) or self._c.recv() != "ready":
                raise RuntimeError("clock sampler did not start")
        except Exception:
            self._p = None
        return self

    def stop(self):
        samples, reasons, max_mhz = [], [], None
        if self._p is not None:
            try:
                self._c.send("stop")
                if self._c.poll(30):
                    samples, reasons, max_mhz = self._c.recv()
            except Exception:
                pass
            self._p.join(timeout=30)
        s = sorted(samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": max_mhz, "reasons": reasons, "samples": len(s),
                "sampler": "NVML, separate process, every 5 ms"}


def algorithmic_bytes(work, n):
    """Bytes the implemented algorithm must move per launch (DESIGN.md §7 per-unit table),
    from the exact work counters of an instrumented run (a pure function of the graph).

    sw = state-word bytes (1 while colours <= 127); WE = 16-B worklist entry; plane = 1-B
    forbidden-colour byte; RED = 4-B atomic on the word holding a plane byte.
      ingest   per vertex : row_ptr 8 + split 4 + sw + plane 1 + one col_idx sector (32)
      Phase A  dense, per vertex swept   : sw + plane 1
               sparse, per entry         : WE 16 + plane 1
               per pending vertex        : sw (tentative colour written)
               per fallback neighbour    : col 4 + sw
      Phase B  dense, per vertex swept   : sw;  per pending vertex : row_ptr 8 + split 4
               sparse, per entry         : WE 16 + sw
               per examined position     : col 4 + sw
               per vertex (commit, once) : sw;  per pushed loser : WE 16
               per scatter edge          : col 4 + RED 4 (counted as scatter_reds, which equals
                                           commit_scatter unless gc_tuning.scatter_filter)
      finalize per vertex : sw + colour 4
    """
    sw = int(work.get("state_bytes") or 1)
    dense_b_pending = work["phase_b_vertices"] - work["sparse_b_entries"]
    return ((8 + 4 + sw + 1 + 32) * n
            + (sw + 1) * work["dense_a_swept"] + 17 * work["sparse_a_entries"]
            + sw * work["phase_a_vertices"] + (4 + sw) * work["phase_a_edges"]
            + sw * work["dense_b_swept"] + 12 * dense_b_pending + (16 + sw) * work["sparse_b_entries"]
            + (4 + sw) * work["phase_b_edges"] + sw * n + 16 * work["pushes"]
            + 8 * work.get("scatter_reds", work["commit_scatter"])
            + (sw + 4) * n)


def survey_bytes(work, n, m):
    """SURVEY §8(d) algorithmic bytes of the method (pull formulation, 4-B gathers):
    B_alg = sum_r [ sum_{v in W_r} (24 + 8 deg v) + sum_{v in W_r} (28 + 8 s_B(v)) ]
    units from the exact counters: sum_r |W_r| = phase_b_vertices, sum_r sum_{v in W_r} deg v
    = m (round 1, W_1 = V) + pending_degree_sum (rounds >= 2), sum s_B = phase_b_edges (the
    positions the conflict scans examine up to their early exit, in this design's scan order)."""
    return (52 * work["phase_b_vertices"] + 8 * (m + work["pending_degree_sum"])
            + 8 * work["phase_b_edges"])


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_record(cfg):
    """ncu numbers of the persistent kernel for this config from profiles/ncu_traffic.json
    (written by scripts/ncu_record.py from an `ncu --set full` capture, stamped with the
    commit it profiled)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f)
    except Exception:
        return None
    r = rec.get("configs", {}).get(cfg)
    if r is None:
        return None
    return dict(r, commit=rec.get("commit"))


def git_commit():
    try:
        import subprocess
        return subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                              text=True, timeout=10).stdout.strip() or None
    except Exception:
        return None


GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
RMAT_CFG = {"rmat16": (16, 8), "rmat24": (24, 16), "rmat27": (27, 16)}


def golden(cfg, policy):
    """The oracle's result for this workload (tests/golden, written by scripts/make_goldens.py,
    which calls only oracle/)."""
    try:
        with open(os.path.join(GOLDEN_DIR, f"oracle_{cfg}_{policy}.json")) as f:
            return json.load(f)
    except Exception:
        return None


def colour_sha(c_u32):
    import hashlib

    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(c_u32, dtype="<u4").tobytes()).hexdigest()


def device_graph(cfg, device):
    """(row_ptr, col_idx) of a BASELINE config on `device` (R-MAT built on the GPU: identical
    to the CPU generator, tests/test_workloads.py)."""
    import torch

    import workloads as wl
    if cfg in RMAT_CFG:
        s, ef = RMAT_CFG[cfg]
        return wl.rmat_range_gpu(s, ef, 0, 1 << s, device=device)
    g = wl.config_graph(cfg)
    return torch.from_numpy(g.row_ptr).to(device), torch.from_numpy(g.col_idx).to(device)


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import oracle  # noqa: F401  (the reference arm is the CPU oracle)
    g, desc = sample_graph(args.config)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.sgr(g)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = g.m / (ms / 1e3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.config, "sample": desc, "n": g.n, "m": g.m, "policy": "higher_id"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{desc}: n={g.n} m={g.m}, oracle_sgr single-threaded C, mean of {args.steps} "
                                   "(warm-up steps not repeated: the oracle keeps no state)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_partitioned(args, rank, world, local):
    """N > 1: one vertex range per rank, one persistent kernel per GPU with the device-initiated
    exchange (include/gc_dist.h); torch.distributed only broadcasts the NCCL id and gathers the
    colours for the parity check after the timed region."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1606_06025_b200 as gc
    import paper_1606_06025_b200.dist as gd
    import workloads as wl

    dev = torch.device("cuda", local)
    if args.config in RMAT_CFG:
        # each rank builds only its own rows on its GPU; ranges uniform in vertex id (the seeded
        # relabelling spreads the degrees evenly: edge imbalance reported below)
        s, ef = RMAT_CFG[args.config]
        n = 1 << s
        bounds = [n * k // world for k in range(world + 1)]
        b, e = bounds[rank], bounds[rank + 1]
        rpl, cil = wl.rmat_range_gpu(s, ef, b, e, device=dev)
        partition = "uniform vertex ranges (seeded relabelling)"
    else:
        g = wl.config_graph(args.config)
        n = g.n
        bounds = [int(x) for x in gc.partition_edge_balanced(g.row_ptr, world)]
        b, e = bounds[rank], bounds[rank + 1]
        rpl, cil = gd.local_slice(g.row_ptr, g.col_idx, b, e)
        rpl, cil = torch.from_numpy(rpl.copy()).to(dev), torch.from_numpy(cil.copy()).to(dev)
        partition = "edge-balanced vertex ranges"
    m_local = torch.tensor([int(rpl[-1])], device=dev, dtype=torch.int64)
    ms_all = [torch.zeros_like(m_local) for _ in range(world)]
    dist.all_gather(ms_all, m_local)
    m_ranks = [int(x.item()) for x in ms_all]
    m = sum(m_ranks)
    comm = gd.init_from_torch(local)
    out = torch.empty(max(e - b, 1), dtype=torch.int32, device=dev)
    kw = dict(policy=args.policy, validate=False, out=out)
    for _ in range(args.warmup):
        gd.color_dist(comm, n, b, e, rpl, cil, **kw)
    clocks = ClockSampler(local).start()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    kms = []
    for _ in range(args.steps):
        r = gd.color_dist(comm, n, b, e, rpl, cil, time_kernel=True, **kw)
        kms.append(r.kernel_ms)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps, sum(kms) / len(kms)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kernel_ms = float(t[0]), float(t[1])
    res = gd.color_dist(comm, n, b, e, rpl, cil, trace=True, **kw)
    # e2e: the same call with this rank's rows and colours in pinned HOST memory
    e2e = None
    if not args.no_e2e:
        h_rp, h_ci = rpl.cpu().pin_memory(), cil.cpu().pin_memory()
        h_out = torch.empty(max(e - b, 1), dtype=torch.int32).pin_memory()
        gd.color_dist(comm, n, b, e, h_rp.numpy(), h_ci.numpy(), policy=args.policy, validate=False,
                      out=h_out.numpy().view(np.uint32))
        dist.barrier()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 5))
        for _ in range(e2e_steps):
            gd.color_dist(comm, n, b, e, h_rp.numpy(), h_ci.numpy(), policy=args.policy, validate=False,
                          out=h_out.numpy().view(np.uint32))
        dist.barrier()
        te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device=dev, dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": m / float(te[0]) / 1e9, "unit": UNIT, "ms_per_step": float(te[0]) * 1e3,
               "h2d_bytes_per_step": 8 * (n + world) + 4 * m, "d2h_bytes_per_step": 4 * n,
               "timing": "host wall clock between barriers, max over ranks (every call is synchronous)"}
    # parity after the timed region: gather the colour ranges to rank 0
    sizes = [bounds[k + 1] - bounds[k] for k in range(world)]
    mx = max(sizes)
    mine = torch.zeros(mx, dtype=torch.int32, device=dev)
    mine[:e - b] = out[:e - b]
    allc = [torch.zeros(mx, dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(allc, mine)
    parity = {}
    if rank == 0:
        colors = np.concatenate([allc[k][:sizes[k]].cpu().numpy().view(np.uint32) for k in range(world)])
        gdn = golden(args.config, args.policy)
        parity["bit_exact_vs_oracle"] = (None if gdn is None else
                                         bool(colour_sha(colors) == gdn["sha256_colors_u32le"]
                                              and res.rounds == gdn["rounds"] and res.num_colors == gdn["num_colors"]
                                              and res.trace == gdn["trace"]))
        if args.config != "rmat27":  # one-GPU reference run on rank 0's GPU
            rp1, ci1 = device_graph(args.config, dev)
            one = gc.color(rp1, ci1, policy=args.policy, validate=False)
            parity["bit_exact_vs_1gpu"] = bool(np.array_equal(one.colors.cpu().numpy().view(np.uint32), colors)
                                               and one.rounds == res.rounds and one.num_colors == res.num_colors)
            del rp1, ci1
    comm.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": m / (ms / 1e3) / 1e9, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": args.config, "n": n, "m": m, "policy": args.policy,
                       "parallelism": f"{partition} x{world}: one persistent kernel per GPU, device-initiated "
                                      "exchange over NVLink peer memory (include/gc_dist.h)",
                       "edge_imbalance": max(m_ranks) / (m / world) - 1.0,
                       "l2": "inputs larger than L2; no flush"},
            "num_colors": res.num_colors, "rounds": res.rounds, **parity,
            "kernel_ms_max_over_ranks": kernel_ms,
            "timing": "CUDA events on each rank's stream around the timed steps, max over ranks",
            "e2e": e2e,
            "gpu_launches": args.steps * 1,  # per step and rank: the persistent kernel
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch

    import paper_1606_06025_b200 as gc

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            return run_partitioned(args, rank, world, local)
        finally:
            dist.destroy_process_group()

    rp, ci = device_graph(args.config, torch.device("cuda", local))
    n, m = int(rp.shape[0]) - 1, int(rp[-1])
    out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    kw = dict(policy=args.policy, validate=False, out=out)

    # untimed instrumented run: exact work counters -> algorithmic bytes per launch
    wres = gc.color(rp, ci, count_work=True, trace=True, **kw)
    work = wres.work
    design_bytes = algorithmic_bytes(work, n)
    alg_bytes = survey_bytes(work, n, m)
    verified = gc.verify(rp, ci, out) == -1
    c = out[:n].cpu().numpy().view(np.uint32)
    gdn = golden(args.config, args.policy)
    bit_exact = (None if gdn is None else
                 bool(colour_sha(c) == gdn["sha256_colors_u32le"] and wres.rounds == gdn["rounds"]
                      and wres.num_colors == gdn["num_colors"] and wres.trace == gdn["trace"]))

    for _ in range(args.warmup):
        gc.color(rp, ci, **kw)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local).start()
    torch.cuda.synchronize()
    e0.record(stream)
    kms = []
    for _ in range(args.steps):
        r = gc.color(rp, ci, time_kernel=True, **kw)
        kms.append(r.kernel_ms)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    kernel_ms = sum(kms) / len(kms)
    value = m / (ms / 1e3) / 1e9

    # e2e: the same call with pinned HOST buffers (H2D of the CSR and D2H of the colours
    # inside the timed region, done by the library)
    e2e = None
    if not args.no_e2e:
        h_rp = rp.cpu().pin_memory()
        h_ci = ci.cpu().pin_memory()
        h_out = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
        h_rp_np, h_ci_np, h_out_np = h_rp.numpy(), h_ci.numpy(), h_out.numpy().view(np.uint32)
        e2e_steps = max(1, min(args.steps, 10))
        gc.color(h_rp_np, h_ci_np, policy=args.policy, validate=False, out=h_out_np)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            gc.color(h_rp_np, h_ci_np, policy=args.policy, validate=False, out=h_out_np)
        e2e_ms = 1e3 * (time.perf_counter() - t0) / e2e_steps
        assert np.array_equal(h_out_np[:n], c)
        e2e = {"value": m / (e2e_ms / 1e3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * (n + 1) + 4 * m, "d2h_bytes_per_step": 4 * n + 224}
        del h_rp, h_ci

    peaks, src = measured_peaks()
    peak = float(peaks["hbm_gbs"])
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    achieved_design = design_bytes / (kernel_ms / 1e3) / 1e9
    nrec = ncu_record(args.config)

    cpu = None
    if not args.no_cpu:
        cpu = cpu_oracle_gteps(args.config)
    if args.cpu_full:  # the oracle on the bench graph itself (minutes at s24)
        import oracle
        import workloads as wl
        g = wl.config_graph(args.config)
        t0 = time.perf_counter()
        cf, _, _ = oracle.sgr(g, args.policy)
        dtf = time.perf_counter() - t0
        cpu = dict(cpu or {}, full_graph={"value": g.m / dtf / 1e9, "unit": UNIT, "seconds": dtf, "cores": 1,
                                          "bit_exact": bool(np.array_equal(cf, c))})

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u%d" % (8 * int(work.get("state_bytes") or 4)),
        "data": "synthetic",
        "config": {"workload": args.config, "n": n, "m": m, "policy": args.policy,
                   "validate": False, "parallelism": "1gpu",
                   "l2": "inputs larger than L2 (CSR %.2f GB > 126 MB); no flush" % ((8 * (n + 1) + 4 * m) / 1e9)},
        "num_colors": wres.num_colors, "rounds": wres.rounds, "verified_ff_fixpoint": verified,
        "bit_exact_vs_oracle": bit_exact,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": nrec.get("dram_bytes") if nrec else None,
                     "traffic_commit": nrec.get("commit") if nrec else None,
                     "peak_source": f"{src} hbm_gbs", "kernel": "sgr_persistent",
                     "kernel_ms": kernel_ms,
                     "alg_bytes_per_launch": alg_bytes,
                     "alg_bytes_model": "SURVEY 8(d): sum_r sum_{v in W_r} (24 + 8 deg v) + (28 + 8 s_B(v)), "
                                        "exact unit counts of this launch (s_B in this design's scan order)",
                     "design_bytes_per_launch": design_bytes,
                     "design_bytes_frac": achieved_design / peak,
                     "ncu_dram_frac": (nrec["dram_bytes"] / (nrec["kernel_ms"] / 1e3) / 1e9 / peak) if nrec else None,
                     "ncu": nrec},
        "work": work,
        "cpu_baseline": cpu,
        "e2e": e2e,
        # per step: the persistent kernel (the variant choice comes from the previous call)
        "gpu_launches": args.steps,
        "clocks": clk,
        "commit": git_commit(),
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--policy", default="higher_id")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-full", action="store_true", help="also time the oracle on the bench graph itself")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""bench.py -- SaCD full sweeps/s (all modes) on B200, through libsacd's C ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--precision f64]
    python bench.py --impl reference ...       (the fp64 CPU oracle on the host cores)

A "step" is one SaCD sweep (U, V and W mode updates: MTTKRP, Gram-Hadamard H, the fused
column-wise SaCD row update, Gram refresh, objective) over the whole synthetic tensor of
the configuration (BASELINE.json configs; default c4, the largest single-GPU one and the
one the north star's scaling target names).  Inputs (the mode-sorted layouts: 3.6 GB for
c4) are larger than the 126 MB L2, so no L2 flush is needed between sweeps.

Prints ONE JSON line on rank 0 (see DESIGN.md section 7 for every field).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "SaCD full sweeps/sec (all modes) on sparse 3-way NTF"
UNIT = "sweeps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="sacd", choices=["sacd", "reference"])
    p.add_argument("--config", default="c4")
    p.add_argument("--rank", type=int, default=None, help="override R (c5 rank sweep)")
    p.add_argument("--precision", default="f64", choices=["f64", "f32"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--reps", type=int, default=5, help="SURVEY 8(d): repetitions with a fresh sacd_init (N = 1)")
    p.add_argument("--nnz-per-item", type=int, default=0)
    p.add_argument("--exchange", default="p2p", choices=["full", "delta", "p2p"],
                   help="N > 1: factor-row exchange of the sharded engine: p2p = changed 16-byte chunks stored "
                        "into the peers' replicas by a kernel over NVLink (CUDA IPC), device flags, graph-captured; "
                        "delta = NCCL (index, value) lists (SURVEY f2); full = NCCL all-gather-v of the owned rows")
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 50 ms while running."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- algorithmic bytes
def algorithmic_bytes(cfg_dims, nnz, R, s):
    """SURVEY 8(d)'s compulsory bytes, with s-byte factor / z_prev elements (s = 8 in the fp64
    build) and Rp = 4 ceil(R/4):
      MTTKRP of mode n : 12 nnz (idx_a, idx_b, val) + 4 (I_n + 1) (row_ptr)
                         + (I_a + I_b) Rp s (every other-factor row once)      -- no M write:
                         8(d) counts M as kept on chip (the fused design);
      row update n     : 2 I_n Rp s (own factor read + write) + 2 I_n R s (z_prev read + write);
      B_comp per sweep : the sum of both over the three modes."""
    d = cfg_dims
    Rp = 4 * ((R + 3) // 4)
    out = {}
    for n in range(3):
        a, b = [m for m in range(3) if m != n]
        mt = 12 * nnz + 4 * (d[n] + 1) + (d[a] + d[b]) * Rp * s
        rows = 2 * d[n] * Rp * s + 2 * d[n] * R * s
        out[n] = (mt, rows)
    bcomp = sum(out[n][0] + out[n][1] for n in range(3))
    return out, bcomp


# ----------------------------------------------------------------------------- oracle (CPU) leg
class OracleSweepSample:
    """The fp64 oracle's sweep (oracle.sacd_run, as it stands) on a bounded sample.

    Per sweep, ora_sacd_run does, for each mode n: the Grams of the two other factors, their
    Hadamard product, the MTTKRP of every row of mode n over its full slice, and the row pass.
    It then does the three Grams for the objective, so every factor's Gram runs three times.
    A step runs exactly those oracle functions on samples and models the full sweep from
    them (calibrated on the GPU box, profiles/r02_oracle_slice_cost.txt):
      * MTTKRP.  The rows of each mode are stratified by slice length (classes
        [2^j, 2^(j+1))).  In every class a systematic sample of rows, with their full slices,
        gets the oracle's mttkrp_layout.  A slice longer than `cap` nonzeros is timed on its
        first `cap` nonzeros and scaled by length: its cost per nonzero does not depend on the
        length.  ora_mttkrp hands rows to threads in chunks of 64 consecutive rows (dynamic), so
        the mode takes max(total CPU time / threads, its heaviest chunk), every row's time
        coming from its class's measured cost per nonzero; the Zipf heads (the first chunks)
        make the second term bind (profiles/r02_oracle_breakdown_c4.txt).
      * Gram.  One full-length strided pass per column pair, over a row subset of at least
        128 MB (every k-th row; smaller subsets stay in cache and run too fast), scaled by k,
        x 3 per factor.
      * Row pass.  Cost per row is independent of the data: every `rstep`-th row, scaled by the
        row share.
    Layouts of the samples are built untimed in the constructor.  step_seconds() returns
    (seconds actually spent, modelled full-sweep seconds)."""

    def __init__(self, c, v, dims, R, seed, budget=3_000_000, rstep=None, cap=1 << 20, gram_bytes=128 << 20):
        import oracle as O
        O.build()
        self.O, self.dims, self.R = O, dims, R
        F = O.init_factors(dims, R, seed)
        self.F = F
        self.cap = cap
        self.rstep = rstep or max(1, int(round(sum(dims) / 100_000)))
        self.strata = []   # (mode, a, b, weight, layout, class, nonzeros of the sampled rows (full length), length scale)
        self.row_len, self.row_cls = [], []
        self.nnz = len(v)
        self.nnz_s = 0
        for n in range(3):
            a, b = O.other_modes(dims, n)
            ci = c[:, n].astype(np.int64)
            ln = np.bincount(ci, minlength=dims[n])
            cls = np.where(ln > 0, np.floor(np.log2(np.maximum(ln, 1))).astype(np.int64), -1)
            classes = [k for k in np.unique(cls) if k >= 0]
            self.row_len.append(ln)
            self.row_cls.append(cls)
            per = budget / max(1, len(classes))
            pick = np.zeros(dims[n], np.int64)   # stratum id + 1 of each sampled row, 0 = not sampled
            info = []
            for j, k in enumerate(classes):
                rows = np.nonzero(cls == k)[0]
                step = max(1, int(np.ceil(ln[rows].sum() / per)))
                sel = rows[::step]
                pick[sel] = j + 1
                info.append((len(rows) / len(sel), sel))
            take = pick[ci] > 0
            cs, vs, st = c[take], v[take], pick[ci[take]] - 1
            for j, (w, sel) in enumerate(info):
                m = st == j
                cj, vj = cs[m].copy(), vs[m]
                remap = np.full(dims[n], -1, np.int64)
                remap[sel] = np.arange(len(sel))
                cj[:, n] = remap[cj[:, n]]
                d2 = list(dims)
                d2[n] = len(sel)
                ia, ib, vv, rp = O.layout(cj, vj, d2, n)
                ln_s = np.diff(rp)
                nz_full = float(ln_s.sum())
                scale = 1.0
                if ln_s.max(initial=0) > cap:
                    keep = np.concatenate([np.arange(rp[i], rp[i] + min(ln_s[i], cap)) for i in range(len(ln_s))])
                    rp2 = np.concatenate([[0], np.cumsum(np.minimum(ln_s, cap))]).astype(np.int64)
                    scale = float(ln_s.sum()) / float(rp2[-1])
                    ia, ib, vv, rp = (np.ascontiguousarray(ia[keep]), np.ascontiguousarray(ib[keep]),
                                      np.ascontiguousarray(vv[keep]), rp2)
                self.strata.append((n, a, b, w, (ia, ib, vv, rp), int(classes[j]), nz_full, scale))
                self.nnz_s += int(rp[-1])
        self.rows = []
        for n in range(3):
            a, b = O.other_modes(dims, n)
            H = O.hadamard(O.gram(F[a]), O.gram(F[b]))
            Fs = np.ascontiguousarray(F[n][::self.rstep])
            self.rows.append((H, Fs, np.zeros_like(Fs)))
        self.gk = [max(1, int(dims[n] * R * 8 // gram_bytes)) for n in range(3)]
        self.gF = [np.ascontiguousarray(F[n][::self.gk[n]]) for n in range(3)]

    def step_seconds(self):
        O = self.O
        T = O.max_threads()
        spent, full = 0.0, 0.0
        cpn = [dict(), dict(), dict()]   # CPU seconds per nonzero, per slice-length class
        for n, a, b, w, (ia, ib, vv, rp), k, nz_full, scale in self.strata:
            t0 = time.perf_counter()
            O.mttkrp_layout(rp, ia, ib, vv, self.F[a], self.F[b])
            dt = time.perf_counter() - t0
            spent += dt
            p = min(T, max(1, (len(rp) - 1 + 63) // 64))   # threads the sample's rows ran on
            cpn[n][k] = dt * p * scale / max(nz_full, 1.0)
        for n in range(3):
            # every row's CPU time from its class's cost per nonzero; ora_mttkrp hands out chunks
            # of 64 consecutive rows (schedule(dynamic, 64)), so the mode takes at least its
            # heaviest chunk -- the Zipf heads sit in the first chunks (c4's W: 15 s of 16)
            ln, cls = self.row_len[n], self.row_cls[n]
            cost = np.zeros(len(ln))
            for k, v in cpn[n].items():
                cost[cls == k] = v
            row_t = ln * cost
            pad = (-len(row_t)) % 64
            chunk_t = np.concatenate([row_t, np.zeros(pad)]).reshape(-1, 64).sum(axis=1)
            full += max(float(row_t.sum()) / T, float(chunk_t.max()))
        for n in range(3):
            H, Fs, M = self.rows[n]
            t0 = time.perf_counter()
            O.mode_pass(M, H, Fs, np.zeros_like(Fs), O.BR_FIRST)
            dt = time.perf_counter() - t0
            spent += dt
            full += dt * (self.dims[n] / len(Fs))
            t0 = time.perf_counter()
            O.gram(self.gF[n])
            dt = time.perf_counter() - t0
            spent += dt
            full += 3.0 * dt * self.gk[n]
        return spent, full

    def describe(self):
        return (f"oracle sweep functions as they stand: mttkrp_layout on slice-length-stratified row samples "
                f"({len(self.strata)} strata, {self.nnz_s} of 3x{self.nnz} slice nonzeros; slices longer than "
                f"{self.cap} timed on their first {self.cap} and scaled by length; per mode max(CPU time / threads, "
                f"heaviest 64-row chunk)) + mode_pass on every {self.rstep}th row + one gram per factor on every "
                f"{self.gk}-th row (>= 128 MB, x k x 3); sample layouts built untimed")


def cpu_baseline(c, v, dims, R, seed, nnz, reps=3):
    import oracle as O
    smp = OracleSweepSample(c, v, dims, R, seed)
    res = [smp.step_seconds() for _ in range(reps)]
    full = float(np.median([r[1] for r in res]))
    spent = float(np.median([r[0] for r in res]))
    out = {"value": 1.0 / full, "unit": UNIT, "cores": O.max_threads(), "kind": "oracle",
           "sample": smp.describe() + f"; median of {reps}", "seconds_per_sweep": full,
           "sample_seconds": spent}
    try:  # the committed full-sweep measurement of the same oracle (tools/oracle_timing.py)
        for ln in open(os.path.join(ROOT, "profiles", "r02_oracle_full_sweeps.jsonl")):
            r = json.loads(ln)
            if r.get("config") == _cfg_name_for(dims) and r.get("rank") == R and r.get("threads") == r.get("host_cores"):
                out["measured_full_sweep"] = {"seconds_per_sweep": r["seconds_per_sweep"], "threads": r["threads"],
                                              "source": "profiles/r02_oracle_full_sweeps.jsonl"}
    except (OSError, ValueError):
        pass
    return out


def measured_gather_peak():
    """Best row-gather rate of the production transport (ldg kernels) on the L1-resident
    table in profiles/r02_gather_bench.jsonl (tools/gather_bench.cu, one B200)."""
    best = None
    try:
        for ln in open(os.path.join(ROOT, "profiles", "r02_gather_bench.jsonl")):
            if not ln.startswith('{"table"'):
                continue
            r = json.loads(ln)
            if r["table"].startswith("L1") and r["kernel"].startswith("ldg"):
                best = max(best or 0.0, r["row_GBps"])
    except (OSError, ValueError, KeyError):
        return None, None
    return best, ("measured: tools/gather_bench.cu ldg transport on an L1-resident 512-byte-row table "
                  "(profiles/r02_gather_bench.jsonl)")


def _cfg_name_for(dims):
    import sacd_inputs as SI
    for k, cfg in SI.CONFIGS.items():
        if tuple(cfg.dims) == tuple(dims):
            return k
    return None


def run_reference(args, cfg, R):
    """--impl reference: the fp64 oracle on the box's host cores (rank 0 only); each step is
    the bounded row sample of OracleSweepSample (seconds actually spent = ms_per_step), value =
    1 / the estimated full-sweep time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    import oracle as O
    import sacd_inputs as SI
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    c, v = SI.make_tensor(cfg, device=dev)
    c, v = c.cpu().numpy().astype(np.uint32), v.cpu().numpy()
    nnz = len(v)
    smp = OracleSweepSample(c, v, cfg.dims, R, cfg.seed)
    K = args.steps if args.steps is not None else 5
    for _ in range(args.warmup):
        smp.step_seconds()
    res = [smp.step_seconds() for _ in range(K)]
    t_full = float(np.mean([r[1] for r in res]))
    t_step = float(np.mean([r[0] for r in res]))
    val = 1.0 / t_full
    cores = O.max_threads()
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * t_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "dims": list(cfg.dims), "nnz": cfg.nnz, "rank": R,
                       "sweep_fraction_per_step": t_step / t_full,
                       "estimated_seconds_per_full_sweep": t_full},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": smp.describe()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def main():
    args = parse()
    import sacd_inputs as SI
    cfg = SI.CONFIGS[args.config]
    R = args.rank or cfg.rank
    if args.impl == "reference":
        run_reference(args, cfg, R)
        return
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2003_03572_b200 import build
    if rank == 0 or world == 1:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2003_03572_b200.sacd import Sacd, nccl_unique_id

    # sharded engine across the N processes: rank 0 makes the NCCL id, torch.distributed
    # broadcasts it (plumbing only); libsacd owns its own communicator.
    shard_kw = {}
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        shard_kw = dict(world_size=world, world_rank=rank, nccl_id=obj[0], exchange=args.exchange)

    K = args.steps if args.steps is not None else cfg.iters
    W = args.warmup
    s = 8 if args.precision == "f64" else 4

    t_gen = time.perf_counter()
    coords, vals = SI.make_tensor(cfg, device="cuda")
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    nnz = int(vals.shape[0])
    stream = torch.cuda.Stream()

    # ---- device-resident timed region (kernel-class events on the launching stream)
    torch.cuda.synchronize()
    t_init = time.perf_counter()
    g = Sacd(coords, vals, cfg.dims, R, cfg.seed, precision=args.precision, stream=stream.cuda_stream,
             profile=False, nnz_per_item=args.nnz_per_item, device=local, **shard_kw)
    init_s = time.perf_counter() - t_init   # sacd_init from device-resident COO (layouts, init, graph)
    info = g.info()
    g.iterate(W)
    g.sync()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    g.iterate(K)
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    # kernel-class breakdown: K more sweeps launched eagerly with per-class CUDA events on
    # the library stream (the timed region above replays the captured sweep graph)
    g.set_profile(True)
    g.profile_reset()
    g.iterate(K)
    g.sync()
    prof = g.profile_read()
    g.set_profile(False)
    f_final, fit_final = g.fit()
    info_end = g.info()
    st_all = g.stats()
    sweep_ms_dev = [r["ms"] for r in st_all[W:W + K]]  # per-sweep device time (sacd_iter_stats.ms)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = K / (ms_max / 1e3)  # sweeps of the whole tensor per second (work split across the ranks)

    per_mode, bcomp = algorithmic_bytes(cfg.dims, nnz, R, s)
    kc = {k: v for k, v in prof.items()}
    dom = max(kc, key=lambda k: kc[k][0])
    launches = info["kernels_per_sweep"] * K   # counted from the captured sweep graph (NCCL kernels excluded)
    mt_ms = kc["mttkrp"][0] / max(kc["mttkrp"][1], 1)
    mt_bytes = sum(per_mode[n][0] for n in range(3)) / 3
    rows_ms = kc["rows"][0] / max(kc["rows"][1], 1)
    rows_bytes = sum(per_mode[n][1] for n in range(3)) / 3
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tr.get(f"{cfg.name}_R{R}_{args.precision}_mttkrp")
    except Exception:
        pass
    if dom == "rows":
        achieved = rows_bytes / (rows_ms / 1e3) / 1e9
        dom_name, dom_bytes, dom_ms = "k_sacd_rows", rows_bytes, rows_ms
    else:
        achieved = mt_bytes / (mt_ms / 1e3) / 1e9
        dom_name, dom_bytes, dom_ms = "k_mttkrp", mt_bytes, mt_ms
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "algorithmic_bytes_per_launch": dom_bytes,
                "avg_launch_ms": dom_ms, "peak_source": peak_src,
                "sweep_hbm_frac": (bcomp / (ms_max / K / 1e3) / 1e9) / hbm_peak,
                "sweep_hbm_frac_8TBs": (bcomp / (ms_max / K / 1e3) / 1e9) / 8000.0,
                "kernel_ms_per_sweep": {k: v[0] / K for k, v in kc.items()}}
    # The MTTKRP is bound by the L1 data path, not HBM: every nonzero gathers
    # one b-row and every fiber one a-row of R_pad * s bytes through L1, plus its 16-byte
    # record.  Peak = 148 SMs x 128 B/clk x the max SM clock (B200_PROFILING.md unit counts).
    pitch = info["pitch"]
    fib = info.get("fibers", [0, 0, 0])
    if world == 1 and all(f > 0 for f in fib):
        # factor-row bytes the MTTKRP moves through L1 per launch (nnz b-rows + one a-row per
        # fiber), against the MEASURED ceiling of the same transport (tools/gather_bench.cu:
        # random 512-byte rows, index by shuffle, x by shared-memory broadcast, LDG.128 per
        # lane, L1-resident table; profiles/r02_gather_bench.jsonl) and the nominal L1 rate
        gathered = sum((nnz + fib[n]) * pitch * s for n in range(3)) / 3
        l1_nominal = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e9
        gpeak, gsrc = measured_gather_peak()
        ach = gathered / (mt_ms / 1e3) / 1e9
        roofline["l1_gather"] = {"achieved": ach, "peak": gpeak or l1_nominal, "unit": "GB/s",
                                 "frac": ach / (gpeak or l1_nominal), "bytes_per_launch": gathered,
                                 "peak_source": gsrc if gpeak else "nominal 148 SM x 128 B/clk (no measurement)",
                                 "nominal_peak": l1_nominal, "frac_of_nominal": ach / l1_nominal,
                                 "what": "factor-row gathers (nnz + fibers) x R_pad x s per MTTKRP launch through L1"}

    # ---- SURVEY 8(d) protocol: repetitions, each with a fresh sacd_init (N = 1)
    g.close()
    del g
    reps = [{"sweeps_per_s": value, "init_s": init_s}]
    if world == 1 and args.reps > 1:
        for _ in range(args.reps - 1):
            torch.cuda.synchronize()
            t = time.perf_counter()
            gr = Sacd(coords, vals, cfg.dims, R, cfg.seed, precision=args.precision, stream=stream.cuda_stream,
                      nnz_per_item=args.nnz_per_item, device=local)
            ti_ = time.perf_counter() - t
            gr.iterate(W)
            gr.sync()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            gr.iterate(K)
            a1.record(stream)
            a1.synchronize()
            reps.append({"sweeps_per_s": K / (a0.elapsed_time(a1) / 1e3), "init_s": ti_})
            gr.close()
    rv = [r["sweeps_per_s"] for r in reps]
    ri = [r["init_s"] for r in reps]
    repetitions = {"n": len(reps), "sweeps_per_s": {"median": float(np.median(rv)), "min": min(rv), "max": max(rv)},
                   "init_s": {"median": float(np.median(ri)), "min": min(ri), "max": max(ri)},
                   "what": "each repetition: fresh sacd_init (device-resident COO), W warm-up sweeps, K timed "
                           "sweeps (CUDA events); the first one is the headline value"}

    # ---- end to end through the public API with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        hc = coords.cpu().pin_memory()
        hv = vals.cpu().pin_memory()
        # the result is read into pinned host buffers allocated once, outside the timed
        # region, as the inputs are (a serving loop reuses them)
        Fout = [torch.empty((cfg.dims[n], R), dtype=torch.float64).pin_memory().numpy() for n in range(3)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        runs = []
        for _ in range(3 if world == 1 else 1):  # N = 1: the median of 3 end-to-end runs
            if world > 1:  # a fresh NCCL id for the second communicator (ids are single-use)
                obj = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                shard_kw = dict(shard_kw, nccl_id=obj[0])
                dist.barrier()
            t0 = time.perf_counter()
            g2 = Sacd(hc, hv, cfg.dims, R, cfg.seed, precision=args.precision, stream=stream.cuda_stream,
                      nnz_per_item=args.nnz_per_item, device=local, **shard_kw)
            t1 = time.perf_counter()
            g2.iterate(K)
            g2.sync()
            t2 = time.perf_counter()
            Fs = g2.factors(out=Fout)
            t3 = time.perf_counter()
            f2, _ = g2.fit()
            t_e2e = time.perf_counter() - t0
            phases = {"init_h2d_layout_s": t1 - t0, "iterate_s": t2 - t1, "factors_d2h_s": t3 - t2,
                      "fit_s": t_e2e - (t3 - t0)}
            te = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            runs.append((float(te.item()), phases))
            g2.close()
            del g2
        runs.sort(key=lambda r: r[0])
        t_e2e, phases = runs[len(runs) // 2]
        h2d = nnz * 16
        d2h = sum(x.nbytes for x in Fs) + 16
        e2e = {"value": K / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
               "seconds": t_e2e, "phases": phases, "runs_seconds": [r[0] for r in runs],
               "runs_phases": [r[1] for r in runs],
               "what": "sacd_init from pinned host COO (H2D + device layout sort) + sacd_iterate(K) + "
                       "sacd_factors (D2H, all modes, into pinned host buffers allocated once) + sacd_fit; "
                       "bytes per step = totals / K; median of the runs"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(coords.cpu().numpy().astype(np.uint32), vals.cpu().numpy(), cfg.dims, R, cfg.seed,
                               nnz)
        except Exception as ex:  # the baseline must never break the bench line
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": args.precision, "data": "synthetic",
                "config": {"workload": cfg.name, "dims": list(cfg.dims), "nnz": nnz, "rank": R,
                           "parallelism": (f"slice-sharded x{world} (factor exchange: "
                                           + {"delta": "NCCL lists of changed elements, rows when smaller)",
                                              "full": "NCCL all-gather-v of owned rows)",
                                              "p2p": "changed 16-byte chunks, head partials and stats stored "
                                                     "into the peers' memory over NVLink by kernels, device flags; "
                                                     "no NCCL per sweep)"}[args.exchange])
                           if world > 1 else "single GPU",
                           **({"exchange_elems_sent": info_end["delta_elems_sent"],
                               "exchange_elems_full_equiv": info_end["full_elems_equiv"]}
                              if world > 1 and info_end.get("delta_exchange") else {}),
                           "l2": "inputs larger than L2 (16-byte nonzero records of the three modes: %.2f GB > 126 MB), no flush" % (48 * nnz / 1e9),
                           "b_comp_bytes_per_sweep": bcomp, "gen_seconds": t_gen,
                           "mttkrp_items": info["items"], "split_rows": info["split_rows"],
                           "objective_after": f_final, "fit_after": fit_final},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk, "init_s": init_s, "repetitions": repetitions,
                "sweep_ms_device": {"median": float(np.median(sweep_ms_dev)) if sweep_ms_dev else None,
                                    "min": min(sweep_ms_dev) if sweep_ms_dev else None,
                                    "max": max(sweep_ms_dev) if sweep_ms_dev else None,
                                    "what": "sacd_iter_stats.ms of the K timed sweeps (%globaltimer, first kernel "
                                            "of the sweep to the end of its objective kernel)"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

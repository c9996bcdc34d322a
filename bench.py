#!/usr/bin/env python
"""Benchmark of the B200 MRRR hot path (BASELINE.json metric: eigenvector entries/s = k*n/s).

One step = one complete solve (every SURVEY §8(a) row: split, root, perturbation, root bisection,
classification, cluster path, singleton RQI + eigenvectors, W/Z stores) of the workload on device.

    python bench.py                          # N=1, C2 (random n=8192, all pairs)
    python bench.py --workload C5a --steps 3
    python bench.py --impl reference         # the CPU oracle timed on this host (reference arm)
    python bench.py --profile sd             # the single/double realisation (mrrr_seig)
    torchrun --nproc-per-node N bench.py --gpus N   # index-range shards, one rank per GPU

Timing: W warm-up steps, then K steps; each step is bracketed by CUDA events on the solver's stream
with an L2 flush (256 MiB write) between steps outside the events; barrier + synchronize around the
timed region; max over ranks.  e2e: the same metric through mrrr_eig_host (host buffers; H2D of d, e
and D2H of W, Z inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import mrrr_inputs as mi  # noqa: E402

METRIC = "eigenvector entries/s (k·n/s), fp64 mixed-prec MRRR all-pairs, 1/2/4/8 B200"
UNIT = "entries/s"


def peaks():
    out = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            out.update(json.load(f))
    except Exception:
        out["hbm_gbs"] = 6650.0
        out["hbm_src"] = "fallback"
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as f:
            out["fp64"] = json.load(f)
    except Exception:
        out["fp64"] = None
    return out


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel_prefix: str, workload: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, median over the captured launches)
    of a kernel from the committed ncu --set full summary of this workload (profiles/ncu_summary_*.json)."""
    import glob
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_summary_*.json"))):
        try:
            js = json.load(open(f))
        except Exception:
            continue
        if js.get("workload") != workload:
            continue
        # a prefix ending in "<" names one kernel exactly (template or not): k_root, not k_root_nodes
        ls = [e for e in js.get("launches", []) if e.get("kernel", "").startswith(kernel_prefix)
              or (kernel_prefix.endswith("<") and e.get("kernel", "") == kernel_prefix[:-1])]
        v = [e["dram_bytes"] for e in ls]
        if v:
            pipe = [e["fp64_pipe_pct"] for e in ls if "fp64_pipe_pct" in e]
            best = (float(np.median(v)), os.path.relpath(f, ROOT) + f" ({len(v)} launches, ncu --set full)",
                    float(np.median(pipe)) if pipe else None)
    return best if best else (None, None, None)


def flush_l2(buf):
    buf.fill_(1.0)  # 256 MiB > 126 MB L2


def reference_arm(args, rank, world):
    """The CPU oracle (oracle/, test infrastructure) timed on this host: the reference arm."""
    if rank != 0:
        return
    import oracle
    cfg = mi.CONFIGS[args.workload]
    d, e = cfg.matrix()
    ksamp = args.ref_k
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.mrrr(d, e, 1, min(8, cfg.n), threads=threads)
    ts = []
    for s in range(args.steps):
        a = 1 + (s * 997) % max(cfg.k - ksamp, 1)
        t0 = time.perf_counter()
        r = oracle.mrrr(d, e, a, a + ksamp - 1, threads=threads, root_side=1)
        ts.append(time.perf_counter() - t0)
        assert r.info == 0
    t = float(np.mean(ts))
    v = ksamp * cfg.n / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+binary128", "data": "synthetic",
            "config": {"workload": args.workload, "n": cfg.n, "k_sample": ksamp, "il_iu": "windows of the C2 index range",
                       "parallelism": "host OpenMP"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{ksamp} eigenpairs per step of {args.workload} (n={cfg.n}), root bisection "
                                       f"of the sample + guards, binary128 RQI"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, d, e, ksamp, sd=False, es=False):
    import oracle
    threads = os.cpu_count() or 1
    oracle.mrrr(d, e, 1, 4, threads=threads, sd=sd, early_stop=es)
    t0 = time.perf_counter()
    r = oracle.mrrr(d, e, 1, ksamp, threads=threads, root_side=1, sd=sd, early_stop=es)
    t = time.perf_counter() - t0
    assert r.info == 0
    return {"value": ksamp * cfg.n / t, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"eigenpairs 1..{ksamp} of {cfg.name} (n={cfg.n}) incl. root bisection of the sample; "
                      f"{t:.2f} s wall on {threads} threads"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C2", choices=sorted(mi.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-k", type=int, default=256)
    ap.add_argument("--cpu-k", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", default="dd", choices=["dd", "sd"],
                    help="dd: fp64 I/O, double-double inside (the headline); sd: the single/double realisation "
                         "(binary32 I/O, binary64 inside, gaptol 1e-5; one GPU)")
    ap.add_argument("--early-stop", action="store_true",
                    help="early classification stop of the root bisection (MRRR_EARLY_STOP, S5', P:3204-3210, "
                         "DESIGN.md A-41; SURVEY 8(f3)); the oracle legs run the same rule")
    args = ap.parse_args()
    SD = args.profile == "sd"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1401_4950_b200 as mrrr

    # MRRR_BENCH_DIST=gloo: functional check of the N > 1 path with ranks sharing the visible GPUs (the
    # collectives then run on host copies; no performance meaning)
    backend = os.environ.get("MRRR_BENCH_DIST", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend == "gloo" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = mi.CONFIGS[args.workload]
    d_np, e_np = cfg.matrix()
    if SD:
        if world > 1:
            raise SystemExit("--profile sd runs on one GPU")
        d_np, e_np = d_np.astype(np.float32), e_np.astype(np.float32)
    fdt = torch.float32 if SD else torch.float64
    n, k = cfg.n, cfg.k
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    ES = args.early_stop
    solver = mrrr.Solver(device=local, stream=stream.cuda_stream, early_stop=ES)
    d = torch.from_numpy(d_np).to(dev)
    e = torch.from_numpy(e_np).to(dev)
    # shard of the index range: contiguous blocks per rank, first-index group ownership
    from paper_1401_4950_b200 import dist as pd
    if world > 1:
        sl, su = pd.shard_range(cfg.il, cfg.iu, world, rank)
        W = None
        # mrrr_eig_dist bootstraps its own NCCL communicator from one id sent over the torch group
        nccl_ident = pd.nccl_id_broadcast() if backend != "gloo" else None
    else:
        W = torch.empty(k, dtype=fdt, device=dev)
        Zt = torch.empty((k, n), dtype=fdt, device=dev)
    flushbuf = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)

    def step():
        with torch.cuda.stream(stream):
            if world == 1:
                (solver.seig if SD else solver.eig)(d, e, cfg.il, cfg.iu, W=W, Z=Zt)
            elif backend != "gloo":
                # the C-ABI multi-GPU call: shard solve + the eigenvalue all-gather over NCCL inside libmrrr
                # (the only collective); Z stays column-sharded
                solver.eig_dist(d, e, cfg.il, cfg.iu, nccl_ident, rank, world)
            else:
                jlo, jhi, Wl, Zl = solver.eig_shard(d, e, sl, su, cfg.il, cfg.iu)
                pd.allgather_eigenvalues(Wl.cpu(), jlo, jhi, cfg.il, cfg.iu)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st0 = solver.stats()
    launches_per_step = st0["launches"]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = []
    rq_ms, rq_n = 0.0, 0
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush_l2(flushbuf)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            evs.append((a, b))
            tm = solver.times()
            rq_ms += tm["rqi_ms_per_launch"] * tm["rqi_launches"]
            rq_n += int(tm["rqi_launches"])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.sum(times)) / args.steps
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        if backend == "gloo":
            t_local = t_local.cpu()
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    value = k * n / (ms_max * 1e-3)
    stats = solver.stats()
    tphase = solver.times()

    # roofline of the dominant kernel family: algorithmic FP64 flops per launch / CUDA-event launch time.
    # Every FP64 operation is counted at the cost the kernels issue (north_star: divisions weighted by their
    # issue cost: 8 FP64 slots, flops.W_DIV_ISSUE); the survey's __ddiv_rn weighting is printed beside it.
    pk = peaks()
    fp = pk.get("fp64") or {}
    roof, roof_other, roof_step = None, None, None
    if fp:
        from paper_1401_4950_b200 import flops as fl
        wdiv_survey = fp.get("w_div", 13.0)
        peak = fp["fp64_tflops"]
        src = "profiles/fp64_peak_r01.json: measured DFMA rate x 2 on this pool's B200 (burst, all SMs)"
        cands = []
        nrq = max(int(tphase["rqi_launches"]), 1)
        # primary: the single dominant kernel (ncu launch list: the root x-NegCount rounds); secondary: the
        # singleton-RQI family (several kernels, timed as a batch incl. its host syncs)
        if tphase["negcount_launches"]:
            launch_ms = tphase["negcount_ms_per_launch"]
            nl = tphase["negcount_launches"]
            f = fl.negcount_flops(stats, n) / nl
            f_sv = fl.negcount_flops(stats, n, wdiv_survey) / nl
            # segmented rounds need at least two segments of seg_minlen = 512 rows per chain half (mrrr.cu,
            # seg_base_k): below n = 2049 (C1) the root rounds are the unsegmented chains of k_root
            if n >= 2049:
                cands.append(("k_negcount_seg (x-NegCount rounds: segmented root chains; child rounds k_negcount_seg_xg/tma)",
                              "k_negcount", launch_ms, f, f_sv))
            else:
                cands.append(("k_root (x-NegCount rounds: one unsegmented chain per lane, n below the segmenting threshold)",
                              "k_root<", launch_ms, f, f_sv))
        if rq_n:
            launch_ms = rq_ms / rq_n
            f = fl.rqi_flops(stats, n, sd=SD) / nrq
            cands.append(("singleton RQI + eigenvectors (k_twist_lane, k_fixed_chunk, k_zwrite_chunk; k_rqi2 for hand-overs)",
                          "k_fixed_chunk", launch_ms, f, f))
        out = []
        for name, pref, launch_ms, f, f_sv in cands:
            ach = f / (launch_ms * 1e-3) / 1e12
            tr, trs, pipe = ncu_traffic(pref, cfg.name)
            out.append({"bound": "alu", "kernel": name, "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                        "frac": ach / peak, "traffic": tr, "traffic_src": trs, "peak_src": src,
                        "launch_ms": launch_ms, "flops_per_launch": f, "ncu_fp64_pipe_pct": pipe,
                        "frac_survey_wdiv": f_sv / (launch_ms * 1e-3) / 1e12 / peak,
                        "note": "achieved = algorithmic FP64 slots at their issued cost (IEEE division = 8 slots) x 2 "
                                "/ launch time; frac_survey_wdiv weights each division by the measured __ddiv_rn "
                                f"cost (w_div = {wdiv_survey}) instead"})
        roof = out[0] if out else None
        roof_other = out[1:] if len(out) > 1 else None
        # whole-solve roofline as the north_star defines it: the slower of (counted FP64 operations, divisions
        # weighted by their issue cost, at peak) and (the Z bytes at HBM bandwidth), against the step time
        ftot = fl.negcount_flops(stats, n) + fl.rqi_flops(stats, n, sd=SD)
        ftot_sv = fl.negcount_flops(stats, n, wdiv_survey) + fl.rqi_flops(stats, n, sd=SD)
        t_fp = ftot / (peak * 1e12)
        zb = (4.0 if SD else 8.0) * k * n
        t_hbm = zb / (pk.get("hbm_gbs", 6550.0) * 1e9)
        t_bound = max(t_fp, t_hbm)
        roof_step = {"bound": "alu" if t_fp >= t_hbm else "hbm", "flops": ftot, "z_bytes": zb,
                     "t_fp64_ms": t_fp * 1e3, "t_hbm_ms": t_hbm * 1e3, "ms_per_step": ms_max,
                     "frac": t_bound * 1e3 / ms_max,
                     "frac_survey_wdiv": max(ftot_sv / (peak * 1e12), t_hbm) * 1e3 / ms_max,
                     "note": "whole solve: algorithmic FP64 slots at issue cost (x-NegCount shared-tree nodes, RQI "
                             "passes) vs Z write bytes; frac = bound time / measured step time"}
        for r_ in out + [roof_step]:
            if r_["frac"] > 1.0:
                raise SystemExit(f"roofline accounting error: frac {r_['frac']:.3f} > 1 for {r_.get('kernel', 'step')}")

    e2e = None
    if world == 1 and not args.no_e2e:
        import torch as _t
        hd = _t.from_numpy(d_np).pin_memory().numpy()
        he = _t.from_numpy(e_np).pin_memory().numpy()
        tdt = _t.float32 if SD else _t.float64
        hW = _t.empty(k, dtype=tdt).pin_memory().numpy()     # page-locked result buffers
        hZ = _t.empty((k, n), dtype=tdt).pin_memory().numpy()
        hs = mrrr.Solver(device=local, early_stop=ES)
        hs.eig_host(hd, he, cfg.il, cfg.iu, W=hW, Zt=hZ, single=SD)
        t0 = time.perf_counter()
        reps = max(1, min(args.steps, 3))
        for _ in range(reps):
            Wh, Zh = hs.eig_host(hd, he, cfg.il, cfg.iu, W=hW, Zt=hZ, single=SD)
        te = (time.perf_counter() - t0) / reps
        hs.close()
        bw = 4 if SD else 8
        e2e = {"value": k * n / te, "unit": UNIT, "h2d_bytes_per_step": bw * (2 * n - 1),
               "d2h_bytes_per_step": bw * k + bw * k * n, "ms_per_step": te * 1e3,
               "path": f"{'mrrr_seig_host' if SD else 'mrrr_eig_host'}: pinned host d, e in, pinned host W, Z out; "
                       "H2D + solve + D2H timed (wall clock)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, d_np.astype(np.float64), e_np.astype(np.float64), min(args.cpu_k, k), sd=SD, es=ES)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64 (binary32 I/O)" if SD else "f64+dd",
                "data": "synthetic" + (", binary32 copy of the workload's matrix" if SD else ""),
                "config": {"workload": cfg.name, "n": n, "k": k, "il": cfg.il, "iu": cfg.iu, "desc": cfg.note,
                           "parallelism": f"index shards x{world}" if world > 1 else "single GPU",
                           "profile": "single/double (mrrr_seig, P:6224-6248, gaptol 1e-5)" if SD
                           else "double/double-double (mrrr_eig)",
                           "early_stop": ES,
                           "l2": "flushed between steps (256 MiB write, outside the events)"},
                "gpu_launches": int(launches_per_step) * args.steps,
                "phases_ms": tphase, "stats": stats, "roofline": roof, "roofline_other": roof_other, "roofline_step": roof_step,
                "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py -- SPS runs to posterior (Algorithm 2) on the
configs[1] workload of BASELINE.json: German-credit-shaped synthetic binary
logit, n = 1000, k = 25, J = 64 groups x N = 1024 particles per GPU, g = 1/16.

One "step" = one complete adaptive SPS run (all SURVEY §8(a) rows: prior
draws, C phases, resampling, M phases with the fused fp64 log-likelihood,
accounting) through the C ABI on data resident in HBM.  `value` = particle x
observation log-likelihood terms evaluated per second, whole job (all ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: launched by torch.distributed.run, one rank per GPU, group sharding.
Default for N > 1 is the north_star's strong-scaling case: configs[4] at a fixed
P = 2^20 particles (J = 1024 groups x N = 1024, cfg2 data), J / N groups per GPU,
plus a 1-GPU run of the same workload on rank 0 (`strong_ref`, speedup = its
time / the N-GPU time).  --scaling weak: 64 groups x 1024 particles per GPU.
--workload cfg4: configs[3] (n = 1e5, k = 100, J = 1024 x N = 1024) sharded.
--impl reference: the CPU oracle (oracle/, the tier's reference arm) on a
bounded sample of the same workload, on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
WORKLOAD = dict(name="cfg2", n=1000, k=25, C=2, J_per_gpu=64, N=1024, g=1.0 / 16)
WORKLOAD_DESC = ("configs[1]: German-credit-shaped synthetic binary logit, n=1000, k=25 (1 + 3 continuous + 21 "
                 "binary covariates, ~30% positives), J=64 groups x N=1024 particles per GPU, Zellner g=1/16, "
                 "data tempering (paper default), residual resampling, full Algorithm 2 to posterior")
ORACLE_SAMPLE = dict(J=16, N=256)
# FP64 pipe peak measured on this pool's B200s (profiles/r01_fp64_peaks.json: DMMA 37.07 TF,
# 64 FMA/clk/SM at 1.96 GHz; DFMA shares the same pipe).  MEASURED_PEAKS.json carries no FP64 figure.
FP64_PEAK_TFLOPS = 37.07
# FP64-pipe operations per pair of K1's binary epilogue (1 DADD relu-sum,
# 10 table-exp, 1 DADD (1 + e), 1 DMUL product), counted from the SASS of k_loglik_bin_mma.
EPILOGUE_DP_OPS_BINARY = 11.0  # counted DP ops of the implemented epilogue (SURVEY 8(d) ii): exp 9, fma(P, e, P), +relu
# K1 contraction: 4 floor(k/4) covariates on DMMA + (k mod 4 <= 2) DFMAs, i.e. k FMAs per pair for
# k = 25; algorithmic contraction flops per pair = 2 k (C - 1).


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", choices=["auto", "weak", "strong"], default="auto",
                    help="auto: configs[1] at N = 1, strong scaling at 2^20 particles for N > 1")
    ap.add_argument("--particles", type=int, default=1 << 20, help="strong scaling: global particle count")
    ap.add_argument("--workload", choices=["cfg2", "cfg4"], default="cfg2")
    ap.add_argument("--no-strong-ref", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ multi-rank host logic
# (plain functions of (world, args, dist): tests/test_multirank_cpu.py runs them under gloo, world_size 2)
def plan_workload(world, scaling_arg="auto", workload="cfg2", particles=1 << 20):
    """Groups / particles per run and the workload description for `world` ranks.  Returns
    dict(data, J, N, g, scaling, desc); J % world == 0 (rank r owns groups [r J / world, (r + 1) J / world))."""
    import sps_synth

    scaling = scaling_arg if scaling_arg != "auto" else ("weak" if world == 1 else "strong")
    if workload == "cfg4":  # configs[3]: one context over all ranks, 1024 / world groups each
        J, N, g, scaling = 1024, 1024, sps_synth.CONFIGS["cfg4"]["g"], "strong"
        desc = ("configs[3]: large synthetic binary logit, n=100000, k=100 (1 + 30 continuous + 69 binary), "
                f"J=1024 x N=1024 particles group-sharded over {world} GPU(s), g=1/4, full Algorithm 2 to posterior")
        return dict(data="cfg4", J=J, N=N, g=g, scaling=scaling, desc=desc)
    N, g = WORKLOAD["N"], WORKLOAD["g"]
    if scaling == "strong":
        J = max(world, particles // N) // world * world
        desc = (f"configs[4] strong scaling: cfg2 data (n=1000, k=25, g=1/16), P={J * N} particles (J={J} x "
                f"N={N}) fixed in total, {J // world} groups per GPU over {world} GPUs, full Algorithm 2 to posterior")
    else:
        J = WORKLOAD["J_per_gpu"] * world
        desc = WORKLOAD_DESC if world == 1 else (WORKLOAD_DESC + f"; weak scaling: 64 groups per GPU x {world}")
    return dict(data="cfg2", J=J, N=N, g=g, scaling=scaling, desc=desc)


def broadcast_id(dist, rank, make_id):
    """Rank 0 makes a 128-byte communicator id (ncclGetUniqueId), every rank receives it."""
    ids = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    return ids[0]


def max_over_ranks(dist, world, x, device):
    """The job's time: max over ranks of a per-rank float (all_reduce MAX; identity at world = 1)."""
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def _lines(self):
        try:
            return open(self.path).read().splitlines()
        except OSError:
            return []

    def start(self):
        """Start sampling every 50 ms; returns once the first sample is in (nvidia-smi takes a few hundred
        ms to start), so that the timed region that follows is covered from its beginning."""
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.n0 = 0
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.gpu)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        t0 = time.time()
        while not self._lines() and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)

    def mark(self):
        """The timed region starts now: samples taken before are dropped."""
        self.n0 = len(self._lines())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self._lines()
        lines = lines[self.n0:] if len(lines) > self.n0 else lines[-1:]  # (a region shorter than one period)
        for line in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                maxs.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(maxs), "reasons": sorted(reasons),
                "samples": len(sms)}


# ------------------------------------------------------------------ oracle (CPU) arm
def oracle_sample(X, y, cov, seed):
    import oracle

    t0 = time.perf_counter()
    r = oracle.run(X, y, 2, ORACLE_SAMPLE["J"], ORACLE_SAMPLE["N"], seed=seed, prior_mean=np.zeros(X.shape[1]),
                   prior_cov=cov, n_threads=os.cpu_count())
    dt = time.perf_counter() - t0
    assert r["status"] == 0, r["status"]
    return r["pairs"], dt


def oracle_cov(X):
    import oracle

    return oracle.g_prior(X, 2, WORKLOAD["g"])


def sample_desc():
    return (f"oracle/ full Algorithm 2 run on the cfg2 data (n=1000, k=25, g=1/16) with J={ORACLE_SAMPLE['J']} x "
            f"N={ORACLE_SAMPLE['N']} particles (a bounded sample of the J=64 x N=1024 workload), OpenMP over "
            f"particles on {os.cpu_count()} host threads; pairs/s over the whole run")


def run_reference(args, rank, world):
    import sps_synth

    if rank != 0:
        return
    X, y = sps_synth.config_data("cfg2")
    cov = oracle_cov(X)
    for w in range(args.warmup):
        oracle_sample(X, y, cov, seed=100 + w)
    pairs = secs = 0.0
    for s in range(args.steps):
        p, dt = oracle_sample(X, y, cov, seed=1 + s)
        pairs += p
        secs += dt
    v = pairs / secs
    # the same workload description (and scaling mode) as our arm at this N; the oracle runs its bounded
    # sample of it (same data, same g) on the host cores
    plan = plan_workload(world, args.scaling, args.workload, args.particles)
    scaling, wdesc = plan["scaling"], plan["desc"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wdesc, "sample": sample_desc()},
            "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample_desc()},
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    import paper_1304_4333_b200 as sps
    import sps_synth

    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_SHORT"), "the contract needs >= 3 warm-up steps"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        nccl_id = broadcast_id(dist, rank, sps.nccl_unique_id)
    else:
        nccl_id = None

    def barrier():
        if world > 1:
            dist.barrier()

    plan = plan_workload(world, args.scaling, args.workload, args.particles)
    X, y = sps_synth.config_data(plan["data"])
    J, N, g, scaling, wdesc = plan["J"], plan["N"], plan["g"], plan["scaling"], plan["desc"]
    n, k = X.shape
    cov = sps.g_prior(X, 2, g, device=local)
    stream = torch.cuda.Stream(device=dev)
    ctx = sps.Sps(X, y, np.zeros(k), cov, J=J, N=N, seed=1, rank=rank, nranks=world, nccl_id=nccl_id,
                  device=local, stream=stream.cuda_stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    for w in range(args.warmup):
        ctx.reset(seed=10_000 + w)
        ctx.run()

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    clocks.mark()
    times, pairs, launches = [], 0.0, 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    last = None
    for s in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(s))  # L2 flush before every timed step (outside the step's events)
        ev0.record(stream)
        ctx.reset(seed=1 + s)
        last = ctx.run()
        ev1.record(stream)
        stream.synchronize()
        times.append(ev0.elapsed_time(ev1))
        pairs += last["pairs"]
        launches += ctx.counters()["launches"]
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    tot_ms = max_over_ranks(dist, world, sum(times), dev)
    value = pairs / (tot_ms / 1e3)

    # ---- roofline of the dominant kernel (K1) measured inside a real run, events on the ctx stream
    ctx.set_profiling(True)
    ctx.reset(seed=999)
    prof_run = ctx.run()
    cnt = ctx.counters()
    ctx.set_profiling(False)
    k1_avg_ms = cnt["k1_ms"] / max(cnt["k1_launches"], 1)
    pairs_per_launch = cnt["k1_pairs"] / max(cnt["k1_launches"], 1)
    ops_per_pair = 2 * k * (WORKLOAD["C"] - 1) + EPILOGUE_DP_OPS_BINARY  # (cfg4's k = 100: the same epilogue)
    achieved = pairs_per_launch * ops_per_pair / (k1_avg_ms * 1e-3) / 1e12
    # FP64 pipe slots actually issued per pair: k FMA-equivalents (DMMA + remainder DFMA) + epilogue ops
    pipe_tflops = pairs_per_launch * 2 * (k * (WORKLOAD["C"] - 1) + EPILOGUE_DP_OPS_BINARY) / (k1_avg_ms * 1e-3) / 1e12
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "r02_k1_ncu.json")
    if not os.path.exists(tr_path):
        tr_path = os.path.join(ROOT, "profiles", "r01_k1_ncu.json")
    if os.path.exists(tr_path):
        traffic = json.load(open(tr_path)).get("dram_bytes_per_launch")
    k1_share = cnt["k1_ms"] / max(sum(times) / max(len(times), 1), 1e-9)
    breakdown = {k: {"ms": round(v, 3), "n": cnt["cat_n"][k]} for k, v in cnt["cat_ms"].items() if cnt["cat_n"][k]}

    # ---- full-data K1 evaluation (P x n pairs in one launch): the M phase's largest case
    th = torch.randn(ctx.P_local, ctx.d, dtype=torch.float64, device=dev) * 0.3
    out = torch.empty(ctx.P_local, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    for _ in range(3):
        ctx.loglik(th.data_ptr(), ctx.P_local, ctx.d, 0, n, out.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(stream)
    for _ in range(reps):
        ctx.loglik(th.data_ptr(), ctx.P_local, ctx.d, 0, n, out.data_ptr())
    e1.record(stream)
    stream.synchronize()
    full_ms = e0.elapsed_time(e1) / reps
    full_pairs_s = ctx.P_local * n / (full_ms * 1e-3)

    # ---- end to end through the public API with host buffers (create from host arrays, run, report to host)
    e2e = None
    if not args.no_e2e:
        Xp = torch.from_numpy(X).pin_memory().numpy()
        yp = torch.from_numpy(y).pin_memory().numpy()
        h2d = Xp.nbytes + yp.nbytes + 8 * k + 8 * k * k
        barrier()
        torch.cuda.synchronize()
        wall = 0.0
        e2e_pairs = 0.0
        d2h = 0
        for s in range(args.steps):
            id2 = None
            if world > 1:  # every communicator needs its own ncclUniqueId (rank 0 makes it, all receive it)
                id2 = broadcast_id(dist, rank, sps.nccl_unique_id)
            t0 = time.perf_counter()
            c2 = sps.Sps(Xp, yp, np.zeros(k), cov, J=J, N=N, seed=1 + s, rank=rank, nranks=world,
                         nccl_id=id2, device=local)
            r2 = c2.run()
            c2.close()
            wall += time.perf_counter() - t0
            e2e_pairs += r2["pairs"]
            L2 = r2["L"]
            d2h = 4 * 6 * L2 + 8 * 6 + 32  # per-cycle trace + moments + logml
        wt = max_over_ranks(dist, world, wall, dev)
        e2e = {"value": e2e_pairs / wt, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    # ---- strong scaling: the same workload on ONE GPU (rank 0; the other ranks wait at the barrier)
    strong_ref = None
    if world > 1 and scaling == "strong" and not args.no_strong_ref:
        if rank == 0:
            c1 = sps.Sps(X, y, np.zeros(k), cov, J=J, N=N, seed=1, device=local, stream=stream.cuda_stream)
            c1.run()  # warm-up (graphs, plans)
            t1s = []
            for s in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.fill_(float(s))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                c1.reset(seed=1 + s)
                r1 = c1.run()
                e1.record(stream)
                stream.synchronize()
                t1s.append(e0.elapsed_time(e1))
            c1.close()
            ms1 = sum(t1s) / len(t1s)
            strong_ref = {"n_gpus": 1, "ms_per_step": ms1, "speedup": ms1 / (tot_ms / args.steps),
                          "note": "same workload, same seeds, one context on rank 0's GPU (no NCCL)"}
        barrier()

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        p, dt = oracle_sample(X, y, oracle_cov(X), seed=7)
        cpu = {"value": p / dt, "unit": "pairs/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": sample_desc(), "seconds": dt}
        # the oracle at THIS configuration (configs[1] exactly, seed 1), timed on a B200 host by
        # tests/test_gpu_headline.py::test_run_parity_cfg2_full (same trajectory as the GPU run)
        full = os.path.join(ROOT, "profiles", "r02_oracle_cfg2_full.json")
        if os.path.exists(full) and args.workload == "cfg2":
            fj = json.load(open(full))
            cpu["same_config"] = {"value": fj["pairs_per_s"], "unit": "pairs/s", "wall_s": fj["oracle_wall_s"],
                                  "threads": fj["threads"], "cpu_model": fj["cpu_model"],
                                  "source": "profiles/r02_oracle_cfg2_full.json"}
        # one core, configs[0] (the SURVEY 8(d) oracle-timing plan)
        import oracle
        import sps_synth as _syn

        X1, y1 = _syn.config_data("cfg1")
        t0 = time.perf_counter()
        r1 = oracle.run(X1, y1, 2, 4, 128, seed=1, prior_mean=np.zeros(4), prior_cov=oracle.g_prior(X1, 2, 0.25),
                        n_threads=1)
        dt1 = time.perf_counter() - t0
        cpu["cfg1_1core"] = {"value": r1["pairs"] / dt1, "unit": "pairs/s", "wall_s": dt1, "cores": 1}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wdesc, "n": n, "k": k, "C": 2, "J": J, "N": N,
                       "global_particles": J * N, "parallelism": f"group-sharded x{world}" if world > 1 else "1 GPU",
                       "l2": "flushed (256 MiB device write) before every timed step",
                       "wall_s_to_posterior": tot_ms / args.steps / 1e3},
            "clocks": clk,
            "strong_ref": strong_ref,
            "e2e": e2e,
            "gpu_launches": launches,
            # K1's contraction runs on the tensor cores' FP64 (DMMA) subpipe, which B200 shares with
            # the FP64 ALU pipe its epilogue uses: bound by that pipe, against its measured rate
            # (MEASURED_PEAKS.json carries no FP64 figure)
            "roofline": {"bound": "tensor", "kernel": f"k_loglik_bin_mma<{k // 4 if k <= 32 else (k + 3) // 4},{k % 4 if k <= 32 and k % 4 in (1, 2) else 0},2> (K1: fp64 DMMA contraction + fused softplus/product epilogue)",
                         "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "ops_per_pair": ops_per_pair, "k1_avg_ms": k1_avg_ms,
                         "pairs_per_launch": pairs_per_launch, "k1_launches_per_run": cnt["k1_launches"],
                         "k1_share_of_step": k1_share,
                         # three readings of the same K1 time: (i) algorithmic contraction flops
                         # 2k per pair; (ii) `frac` above, 2k flops + the 11 counted epilogue ops per pair;
                         # (iii) FP64-pipe slots, k FMA + 11 epilogue ops per pair against 64 slots / clk / SM
                         # -- what the shared DMMA / DFMA pipe actually enforces
                         "frac_contraction": pairs_per_launch * 2 * k * (WORKLOAD["C"] - 1) / (k1_avg_ms * 1e-3) / 1e12
                         / FP64_PEAK_TFLOPS,
                         "frac_pipe_slots": pipe_tflops / FP64_PEAK_TFLOPS,
                         "peak_source": "measured FP64 DMMA rate, 37.07 TF/s (tools/fp64_peaks.cu, profiles/r01_fp64_peaks.json; "
                                        "the DFMA epilogue shares the pipe); ncu: profiles/r02_k1_ncu.json, profiles/r02_ncu_k1_hot.txt, "
                                        "profiles/r02_ncu_fused_vs_k1.txt",
                         "full_data_eval": {"ms": full_ms, "pairs_per_s": full_pairs_s,
                                            "frac": full_pairs_s * ops_per_pair / 1e12 / FP64_PEAK_TFLOPS}},
            "cpu_baseline": cpu,
            "run": {"logml": last["logml"], "logml_nse": last["logml_nse"], "cycles": last["L"],
                    "m_steps": last["total_m_steps"], "mean": list(last["mean"]), "nse": list(last["nse"]),
                    "pairs_per_run": last["pairs"], "syncs_per_run": cnt["syncs"],
                    "profiled_breakdown_ms": breakdown},
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

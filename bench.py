#!/usr/bin/env python
"""bench.py -- DFLOP plan-candidate evaluation on B200 (contract: DESIGN.md section 8).

One step = one pass of the whole hot path over one synthetic global batch: a1 predict,
a2 order, a3/a4 every candidate of the family (LPT + swap refinement + 1F1B score), a5
argmin (NCCL min all-reduce + broadcast of the winner for N > 1) and the winner's
assignment, through the C-ABI call ``dflop_search_plans``.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl dflop|reference]

N > 1 is launched by torchrun (one rank per GPU).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate plans evaluated/sec and p50 plan latency per global batch, 1/2/4/8 B200"
UNIT = "candidate plans/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, help="BASELINE.json config (1-based)")
    ap.add_argument("--impl", choices=["dflop", "reference"], default="dflop")
    ap.add_argument("--K", type=int, default=0, help="override the family size")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle baseline budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--order4", action="store_true", help="DFLOP_MODE_ORDER4: per-candidate slot-order choice")
    ap.add_argument("--tick-ns", type=float, default=0.0,
                    help="override the preset's integer time unit (1 = nanosecond ticks: the 64-bit kernel variant)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------- workload
def workload(args, world):
    import dataclasses

    from paper_2603_25120_b200 import synth
    p = synth.presets()[args.config]
    if args.tick_ns:
        p = dataclasses.replace(p, model=dict(p.model, tick_ns=float(args.tick_ns)))
    K = args.K or p.K
    if p.plan is None:  # config 4: the Algorithm-1 search (Stage A + P plans x K candidates)
        return p, K, "strong", None, None
    scaling = "strong"
    if p.K_scaling == "weak":
        K = K * world
        scaling = "weak"
    m = p.plan["n_mb"] * p.plan["l_dp"]
    S = p.plan["e_pp"] + p.plan["l_pp"]
    return p, K, scaling, m, S


def algorithmic_ops_per_candidate(n, m, S, R, G):
    """Integer ops the method must execute per candidate:
    LPT n*m probes x 5 ops; refinement R*(n/m)*(n/m+1) pair evaluations x 8 ops;
    1F1B 2*S*m op updates x 4 ops; Philox-4x32-10 draws ceil(n/G)*ceil((G-1)/4) x 80 ops."""
    per = n / max(m, 1)
    lpt = 5.0 * n * m
    ref = 8.0 * R * per * (per + 1)
    sim = 4.0 * 2 * S * m
    philox = 80.0 * (-(-n // G)) * (-(-(G - 1) // 4))
    return lpt + ref + sim + philox


def config_dict(args, p, K, m, S, world):
    """The `config` object of the JSON line -- identical for the GPU arm and the reference arm."""
    return {"workload": p.name, "n": p.n, "m": m, "S": S, "K": K, "K_per_gpu": K // world,
            "plans": p.top_p if p.plan is None else 1, "order4": bool(args.order4), "R": p.R, "G": p.G,
            "plan": p.plan if p.plan is not None else "searched (Algorithm 1 Stage A + Stage B)",
            "tick_ns": p.model["tick_ns"], "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": f"candidate-shard x{world}"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def int_peaks():
    """profiles/int_peaks.json (tools/int_peaks.cu, measured on a B200 of this pool)."""
    f = os.path.join(ROOT, "profiles", "int_peaks.json")
    return json.load(open(f)) if os.path.exists(f) else None


def stage_a_ops_per_pair(model, mem):
    """fp64 arithmetic operations (add/sub/mul/div, one each) of one Stage-A (config, N_mb)
    pair as csrc/stage_a.cu evaluates Algorithm 1 (O9), for the model's
    grid shapes: (memory part, everything after the Eq. (4)-(5) check)."""
    def lerp1d(nx):
        return 0 if nx == 1 else 7                       # w = (x - x_k) / (x_k+1 - x_k); dlerp
    def interp_thr(g):
        l1 = lerp1d(len(g["x"]))
        return l1 if len(g["tp"]) == 1 else 3 + 2 * l1 + 4
    def interp_mem(g):
        l1 = lerp1d(len(g["x"]))
        plane = l1 if len(g["tp"]) == 1 else 3 + 2 * l1 + 4
        return 3 + 2 * plane + 4
    mem_part = 6 + 4 + sum(interp_mem(mem[k]) for k in ("ms_e", "as_e", "ms_l", "as_l"))
    rest = 13 + (1 if model.get("e_attn") else 0) + 1 + 4 + 2 + 3 + 1 + 7 + 2 + \
        interp_thr(model["thr_e"]) + interp_thr(model["thr_att"]) + interp_thr(model["thr_lin"])
    return mem_part, rest


# ---------------------------------------------------------------- clocks (NVML)
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, device: int, period: float = 0.05):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self.period = period
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        names = [v for k, v in REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU oracle baseline
def oracle_rate(p, K_family, budget_s, threads=None):
    """The oracle as it stands, on the host cores: predict + candidates over a bounded sample of
    the same workload (consecutive candidate ranges until ~budget_s of wall time).  Returns
    (candidates/s, sample description, threads used)."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    t, f, x = p.features(0)
    t0 = time.perf_counter()
    plan, what = p.plan, ""
    if plan is None:  # Algorithm 1: the oracle's own Stage A, then the leader plan's family
        mb, msq = O.batch_means(p.model, t, f, x)
        T_A, cfgs = O.stage_a_all(p.model, p.mem(), p.cluster["n_gpus"], p.cluster["gpus_per_node"], p.gbs, mb, msq)
        e, i = O.pair_to_config(cfgs, p.gbs, O.stage_a_top(T_A, 1)[0])
        c = cfgs[e]
        plan = dict(e_tp=int(c[0]), e_pp=int(c[1]), e_dp=int(c[2]), l_tp=int(c[3]), l_pp=int(c[4]), l_dp=int(c[5]),
                    n_mb=i)
        what = " (Stage A over all pairs, then the Stage-A leader plan's family)"
    _, q, st, _ = O.predict(p.model, plan, t, f, x)
    done = 0
    chunk = threads * 8
    while True:
        c1 = min(K_family, done + chunk)
        O.balance_threaded(q, plan, K_family, p.R, p.G, p.seed(0), done, c1, threads=threads, per_candidate=False)
        done = c1
        dt = time.perf_counter() - t0
        if dt >= budget_s or done >= K_family:
            break
        chunk = min(max(chunk, int(done / dt * 2.0)), threads * 4096)
    return (done / dt, f"candidates [0, {done}) of batch 0 (+ predict of all {p.n} samples){what}, {dt:.1f} s",
            threads)


def oracle_rate_1thread(p, K_family, n_cand=1024):
    """BASELINE.md 4.2 / SURVEY 8(d): the oracle on ONE thread over a fixed subset of 1,024
    candidates [0, 1024) of batch 0 (predict excluded): a per-core rate."""
    from oracle import oracle as O
    t, f, x = p.features(0)
    plan = p.plan
    if plan is None:
        return None
    _, q, _, _ = O.predict(p.model, plan, t, f, x)
    c1 = min(K_family, n_cand)
    t0 = time.perf_counter()
    O.balance(q, plan, K_family, p.R, p.G, p.seed(0), 0, c1, per_candidate=False)
    return c1 / (time.perf_counter() - t0), c1


def run_reference(args):
    """The reference arm: the CPU oracle as it stands on the host cores, each step a bounded
    sample of the workload; ms_per_step is the measured wall time of a step."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    p, K, scaling, m, S = workload(args, world)
    threads = os.cpu_count() or 1
    steps, warm = args.steps, args.warmup
    per_step_budget = max(2.0, min(20.0, 150.0 / max(1, steps + warm)))
    rates, walls, samples = [], [], []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        r, sample, thr = oracle_rate(p, K, per_step_budget, threads)
        w = time.perf_counter() - t0
        if i >= warm:
            rates.append(r)
            walls.append(w)
            samples.append(sample)
    value = statistics.mean(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": warm, "ms_per_step": 1e3 * statistics.mean(walls),
        "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config_dict(args, p, K, m, S, world),
        "reference_note": "reference arm = the CPU oracle (no installable reference: the paper ships no code); "
                          "each step evaluates a bounded sample of the family (ms_per_step = its measured wall time)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": f"each step: {samples[-1] if samples else ''}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# The JSON line is the only thing this program writes to stdout: file descriptor 1 is pointed
# at stderr for everything else (NCCL prints its version banner to stdout when NCCL_DEBUG is
# set, and other C libraries may print too); emit() writes to the saved original stdout.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict) -> None:
    _claim_stdout()
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()


# ---------------------------------------------------------------- the GPU arm
def main():
    _claim_stdout()
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_25120_b200 import dflop as D

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    p, K, scaling, m, S = workload(args, world)
    comm = D.Comm(rank, world, dev.index) if world > 1 else None
    n_batches = 8
    host = [p.features(b) for b in range(n_batches)]
    to_dev = lambda a: torch.from_numpy(a.astype(np.uint32).view(np.int32)).to(dev)
    dfeat = [tuple(to_dev(a) for a in h) for h in host]
    ws = D.Workspace()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    alg1 = p.plan is None
    P = p.top_p if alg1 else 1

    def search(t, f, x, b):
        if alg1:  # Algorithm 1: Stage A on the batch, Stage B over the top-P plans
            return D.search_plans_batches(p.model, t, f, x, [0, p.n], K=K, R=p.R, G=p.G, seed=p.seed(b), comm=comm,
                                          cluster=p.cluster, mem=p.mem(), gbs=p.gbs, top_p=P, ws=ws,
                                          order4=args.order4)
        return D.search_plans(p.model, t, f, x, K=K, R=p.R, G=p.G, seed=p.seed(b), plan=p.plan,
                              comm=comm, want_assign=True, ws=ws, order4=args.order4)

    def step(b):
        t, f, x = dfeat[b % n_batches]
        return search(t, f, x, b % n_batches)

    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    # ---- timed region (device time, CUDA events on the launching stream)
    D.profile_read(reset=True)
    D.profile_enable(True)
    times = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            flush.zero_()                       # L2 flushed between timed iterations
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = step(args.warmup + i)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    D.profile_enable(False)
    prof = D.profile_read(reset=True)
    total_ms = sum(times)
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        lat = torch.tensor(times, dtype=torch.float64, device=dev)
        dist.all_reduce(lat, op=dist.ReduceOp.MAX)
        times = lat.tolist()
    value = P * K * args.steps / (total_ms / 1e3)      # whole-job candidates per second
    ms_per_step = total_ms / args.steps
    p50 = statistics.median(times)
    p99 = float(np.percentile(np.array(times), 99))

    # ---- e2e: the public call with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        pinned = [tuple(torch.from_numpy(a.astype(np.uint32).view(np.int32)).pin_memory() for a in h) for h in host]
        dbuf = tuple(torch.empty(p.n, dtype=torch.int32, device=dev) for _ in range(3))
        out_host = torch.empty(p.n, dtype=torch.int32).pin_memory()
        e_times = []
        for i in range(args.warmup + args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for d_, h_ in zip(dbuf, pinned[i % n_batches]):
                d_.copy_(h_, non_blocking=True)
            r = search(*dbuf, i % n_batches)
            out_host.copy_(r["assign"], non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            if i >= args.warmup:
                e_times.append(e0.elapsed_time(e1))
        e_total = sum(e_times)
        if world > 1:
            tt = torch.tensor([e_total], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_total = float(tt.item())
        e2e = {"value": P * K * len(e_times) / (e_total / 1e3), "unit": UNIT, "h2d_bytes_per_step": 3 * 4 * p.n,
               "d2h_bytes_per_step": 4 * p.n + 32 + 8, "p50_ms": statistics.median(e_times)}

    # ---- which candidate-kernel variant ran: k_build_items picks the 64-bit sums when a batch's
    # sum of e or l reaches 2^32 - 1 ticks (the u32 variants' bound on every bucket sum)
    _, tk = D.predict_costs(p.model, p.plan if not alg1 else res["plan"], *dfeat[0], want_f32=False)
    tk = tk.cpu().numpy().view(np.uint32).astype(np.uint64)
    wide_sums = int(tk[0].sum() + tk[1].sum()) >= (1 << 32) - 1 or int(tk[2].sum() + tk[3].sum()) >= (1 << 32) - 1

    # ---- roofline of the dominant kernel (candidates: integer-issue bound)
    b, e = (K * rank) // world, (K * (rank + 1)) // world
    if alg1:
        # P plans of different shapes overlap on the Stage-B streams: their summed algorithmic
        # work over the step's device time (a lower bound of the kernels' own rate)
        plans = res["plans"]
        ops_step = sum(algorithmic_ops_per_candidate(p.n, q["n_mb"] * q["l_dp"], q["e_pp"] + q["l_pp"], p.R, p.G)
                       for q in plans) * (e - b)
        m = sum(q["n_mb"] * q["l_dp"] for q in plans) / max(1, len(plans))
        S = None
        ops_launch, cand_ms = ops_step, ms_per_step
    else:
        ops_launch = algorithmic_ops_per_candidate(p.n, m, S, p.R, p.G) * (e - b)
        cand_ms = prof["cand_ms"] / max(1, prof["cand_launches"])
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    achieved = ops_launch / (cand_ms / 1e3) / 1e12
    ip = int_peaks()
    if ip:
        # measured (tools/int_peaks.cu -> profiles/int_peaks.json): instruction issue with both
        # integer pipes busy (adds split by ptxas over IADD3 / IMAD.IADD), and the ALU pipe alone
        # (IADD3, VIMNMX, VIADDMNMX, LOP3 -- the pipe the LPT probes and min trees run on)
        peak_issue = ip["add_u32_ptxas_choice"]["lane_ops_per_s"] / 1e12
        peak_alu = ip["viaddmnmx_u32"]["lane_ops_per_s"] / 1e12
        note = (f"measured: profiles/int_peaks.json (tools/int_peaks.cu, {ip['gpu']}, "
                f"{ip['add_u32_ptxas_choice']['sm_mhz_in_kernel']} MHz): issue "
                f"{ip['add_u32_ptxas_choice']['lane_ops_per_clk_per_sm']:.1f} lane-ops/clk/SM, ALU pipe "
                f"{ip['viaddmnmx_u32']['lane_ops_per_clk_per_sm']:.1f} lane-ops/clk/SM")
    else:
        sm_max = 1965.0
        peak_issue = n_sm * 4 * 32 * sm_max * 1e6 / 1e12
        peak_alu = peak_issue / 2
        note = "fallback: 148 SM x 4 SMSP x 32 lanes x 1965 MHz (profiles/int_peaks.json missing)"
    variant = "u64" if wide_sums else "u32"
    # the same work without the refinement pairs the windowed search proves irrelevant: on
    # config 5 about 2% of the (i, i') pairs fall in a row's window (DESIGN.md section 6,
    # oracle analysis of batch 0), so the refinement term shrinks to that share
    frac_pruned = None
    if not alg1 and prof.get("split_chunks"):
        per = p.n / max(m, 1)
        ref = 8.0 * p.R * per * (per + 1)
        ops_pruned = (algorithmic_ops_per_candidate(p.n, m, S, p.R, p.G) - 0.98 * ref) * (e - b)
        frac_pruned = ops_pruned / (cand_ms / 1e3) / 1e12
    kname = f"k_candidates<{variant}>"
    if variant == "u32" and prof.get("split_chunks"):  # the host launched the split pipeline
        kname = "k_lpt + k_candidates<u32> (split pipeline, %d chunks per step)" % (prof["split_chunks"] // args.steps)
    roofline = {"bound": "issue", "kernel": kname, "achieved": achieved, "peak": peak_issue,
                "unit": "Tops/s", "frac": achieved / peak_issue, "traffic": None,
                "peak_alu_pipe": peak_alu, "frac_alu_pipe": achieved / peak_alu,
                "kernel_ms": cand_ms, "kernel_share_of_step": cand_ms / ms_per_step,
                "peak_note": note, "ops_per_candidate": ops_launch / max(1, (e - b) * P),
                "ops_note": "nominal work of the method (DESIGN.md section 8); the split pipeline's windowed "
                            "refinement search scores only the pairs that could be applied (about 2% on config 5) "
                            "with the same result -- frac_without_pruned_pairs counts only those, ncu_* give the "
                            "executed-instruction utilisation"}
    if frac_pruned is not None:
        roofline["frac_without_pruned_pairs"] = frac_pruned / peak_issue
    stage_a = None
    if alg1:
        roofline["kernel"] = "k_candidates<u32> x P plans (Stage B, 4 streams)"
        # Stage A alone (k_stage_a, fp64 closed forms over every (config, N_mb) pair), timed by
        # the library's events over the timed steps; roofline against the measured fp64 rate
        if prof.get("stage_a_launches"):
            sa_ms = prof["stage_a_ms"] / prof["stage_a_launches"]
            mem_ops, rest_ops = stage_a_ops_per_pair(p.model, p.mem())
            ops = res["n_pairs"] * mem_ops + res["n_feasible"] * rest_ops
            ach = ops / (sa_ms / 1e3) / 1e12
            stage_a = {"kernel": "k_stage_a", "ms": sa_ms, "pairs": res["n_pairs"], "feasible": res["n_feasible"],
                       "pairs_per_s": res["n_pairs"] / (sa_ms / 1e3), "share_of_step": sa_ms / ms_per_step,
                       "fp64_ops_per_pair": {"memory_check": mem_ops, "durations": rest_ops},
                       "roofline": {"bound": "fp64", "achieved": ach, "unit": "Tops/s"}}
            if ip and "dadd_f64" in ip:
                pk = ip["dadd_f64"]["lane_ops_per_s"] / 1e12
                stage_a["roofline"].update(peak=pk, frac=ach / pk,
                                           peak_note="measured DADD/DMUL lane-ops/s (profiles/int_peaks.json, 64 per "
                                                     "clk per SM); a DDIV counts one algorithmic op but issues a "
                                                     "Newton sequence of ~10 fp64 instructions")
        roofline["duration_note"] = "device step time (Stage A + Stage B)"
    # traffic: dram__bytes_read.sum + dram__bytes_write.sum of the candidate kernel from the
    # committed ncu capture (profiles/traffic.json), per candidate x this launch's K
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        tr = json.load(open(traffic_file)).get(p.name)
        if tr:
            roofline["traffic"] = tr["dram_bytes_per_candidate"] * (e - b)
            roofline["traffic_unit"] = "B"
            roofline["traffic_source"] = tr["source"]
            # the same capture's achieved instruction issue (smsp__issue_active, % of peak):
            # the issue roofline the kernel runs at, beside the algorithmic-op fraction above
            if "ncu_issue_active" in tr:
                roofline["ncu_issue_active"] = tr["ncu_issue_active"]
                for k in ("ncu_lsu_data_pipe_wavefronts", "ncu_alu_pipe", "ncu_per_kernel"):  # the busiest pipes
                    if k in tr:
                        roofline[k] = tr[k]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": variant, "data": "synthetic",
        "config": config_dict(args, p, K, m if not alg1 else None, S, world),
        "p50_plan_latency_ms": p50, "p99_plan_latency_ms": p99,
        "candidate_microbatches_per_s": value * m,
        "e2e": e2e,
        "gpu_launches": int(prof["kernel_launches"]),
        "roofline": roofline,
        "clocks": clk.summary(),
        "winner": {"batch": (args.warmup + args.steps - 1) % n_batches, "cand": res["cand"],
                   "makespan_ticks": res["makespan"], "cmax_ticks": res["cmax"], "plan": res["plan"]},
        "kernel_variant": variant,
        "stage_a": stage_a,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample, thr = oracle_rate(p, K, args.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": thr, "cpu_model": cpu_model(), "kind": "oracle",
                                "sample": sample}
        one = oracle_rate_1thread(p, K)
        if one:
            line["cpu_baseline"]["per_core"] = {"value": one[0], "unit": UNIT, "threads": 1,
                                                "sample": f"candidates [0, {one[1]}) of batch 0, one thread"}
    if rank == 0:
        emit(line)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""bench.py — DFSAttn sparse self-attention path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload HY]

One step = one update-step call of the hot path for ALL heads of one layer at
HunyuanVideo-720p (33x45x80 = 118,800 tokens, 24 heads, d=128, B=128, B_s=16,
gamma=0.1 -> K=93 of M=929 blocks, 90% block sparsity):
  K2 permute Q/K/V (+ fused pooling) -> K3 hierarchical scores -> K4 top-K ->
  K5 block-sparse attention with the unpermute fused into its epilogue.
Inputs are synthetic smooth Gaussian video fields (4 rounds of clamped
6-neighbour averaging, re-standardised), bf16 [N, H, d].
Heads are sharded across ranks (strong scaling of one 24-head call): rank r
owns heads [r*H/P, (r+1)*H/P); no collective on the data path.

value = dense-equivalent TFLOP of the whole call / max-over-ranks time
("effective TFLOPS", BASELINE.json). ms_per_step = ms per call.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {  # SURVEY.md §8 config shorthand
    "HY": dict(dims=(33, 45, 80), heads=24, d=128, gamma=0.1, block=128, sub=16,
               name="HunyuanVideo-720p 129f: 33x45x80=118800 tok, 24 heads, d=128, 90% block sparsity"),
    "W7": dict(dims=(21, 45, 80), heads=40, d=128, gamma=0.1, block=128, sub=16,
               name="Wan2.1-14B 720p: 21x45x80=75600 tok, 40 heads, d=128, 90% block sparsity"),
    "W4": dict(dims=(21, 30, 52), heads=40, d=128, gamma=0.15, block=128, sub=16,
               name="Wan2.1-14B 480p: 21x30x52=32760 tok, 40 heads, d=128, 85% block sparsity"),
    "C": dict(dims=(13, 30, 45), heads=48, d=64, gamma=0.2, block=128, sub=16,
              name="CogVideoX-5B: 13x30x45=17550 tok, 48 heads, d=64, 80% block sparsity"),
}
METRIC = "block-sparse attn effective TFLOPS (dense-equivalent) per call, HunyuanVideo 720p, 90% sparsity"


def metric_for(workload: str, wl: dict | None = None) -> str:
    """BASELINE.json's metric for the headline workload; the other configs name themselves."""
    w = wl or WORKLOADS[workload]
    if workload == "HY" and w["gamma"] == WORKLOADS["HY"]["gamma"]:
        return METRIC
    return f"block-sparse attn effective TFLOPS (dense-equivalent) per call, {w['name']}"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML every 10 ms
    from a thread (nvidia-smi -lms as the fallback when NVML is unavailable)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self.power = []  # W
        self.stop = threading.Event()
        self.proc = None
        self.thread = None

    def _nvml_loop(self, nv, hdl):
        bits = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)))
                try:
                    self.power.append(nv.nvmlDeviceGetPowerUsage(hdl) / 1000.0)
                except Exception:
                    pass
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(hdl)
                self.reasons.update(name for bit, name in bits.items() if r & bit)
            except Exception:
                pass
            self.stop.wait(0.01)

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            hdl = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(hdl, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, hdl), daemon=True)
            self.thread.start()
            return self
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._smi_read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _smi_read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                try:
                    self.sm.append(float(parts[0]))
                    self.max_mhz = float(parts[1])
                    self.power.append(float(parts[2]))
                except ValueError:
                    continue
                self.reasons.update(self.NAMES[i] for i in range(4) if parts[3 + i].lower() == "active")

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        out = {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
               "samples": len(self.sm)}
        if self.power:
            out["power_w"] = round(statistics.median(self.power), 1)
        return out


def smooth_fields(dims, heads, d, seed, device, rounds=4):
    """Three bf16 [N, H, d] smooth Gaussian fields (q, k, v) generated on the GPU
    with torch (input synthesis, not the timed path): the reference's
    gen_video_field recipe (synthetic.cpp:228-284) at device speed."""
    import torch

    f, h, w = dims
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = []
    for _ in range(3):
        x = torch.randn((f, h, w, heads * d), generator=g, device=device, dtype=torch.float32)
        for _ in range(rounds):
            p = torch.nn.functional.pad(x.permute(3, 0, 1, 2).unsqueeze(0), (1, 1, 1, 1, 1, 1), mode="replicate")[0]
            c = p[:, 1:-1, 1:-1, 1:-1]
            s = c + p[:, :-2, 1:-1, 1:-1] + p[:, 2:, 1:-1, 1:-1] + p[:, 1:-1, :-2, 1:-1] + p[:, 1:-1, 2:, 1:-1] \
                + p[:, 1:-1, 1:-1, :-2] + p[:, 1:-1, 1:-1, 2:]
            x = (s / 7.0).permute(1, 2, 3, 0).contiguous()
            del p, c, s
            x = x / x.std()
        out.append(x.reshape(f * h * w, heads, d).to(torch.bfloat16).contiguous())
        del x
    return out


def k5_traffic(workload, heads_local):
    """DRAM bytes (read + write) per K5 launch from the committed ncu --set full capture
    (profiles/<round>/k5_traffic.json), scaled to this rank's head count; None if absent."""
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "k5_traffic.json"))):
        try:
            with open(path) as f:
                rec = json.load(f)
        except (OSError, ValueError):
            continue
        if rec.get("workload") == workload:
            best = rec
    if not best:
        return None
    return best["dram_bytes_per_launch"] * heads_local / best["heads"]


def executed_flops(lut, n, block, d):
    """4*d*sum over (head, u, v in I_u) of r_u*c_v with real token counts."""
    import torch

    m = lut.shape[1]
    sizes = torch.full((m,), block, dtype=torch.float64, device=lut.device)
    sizes[-1] = n - (m - 1) * block
    cols = sizes[lut.long()].sum(-1)  # [H, M]
    return float(4.0 * d * (cols * sizes[None, :]).sum().item())


class RefSampler:
    """The reference's own CPU path (oracle/_ref: the unmodified reference sources) on a
    bounded sample of one call: per head the full reorder + pooled keys (timed
    separately), then `units_per_head` (head, query-block) units of pooled scoring +
    top-K + attend_row over the unit's K blocks, parallel over all host threads with the
    reference's parallel_for. Extrapolated to one H-head call as
        fixed_s * ceil(H / threads) + units_s * (H * M) / units."""

    def __init__(self, wl, threads=None):
        import ctypes as C

        from oracle import ref

        self.C, self.ref = C, ref
        self.dims, self.H, self.d = wl["dims"], wl["heads"], wl["d"]
        self.B, self.Bs, self.gamma = wl["block"], wl["sub"], wl["gamma"]
        self.n = self.dims[0] * self.dims[1] * self.dims[2]
        self.m = -(-self.n // self.B)
        self.threads = threads or os.cpu_count() or 1
        self.heads_s = min(self.H, self.threads)
        if ref is None:
            self.ctx = None
            return
        lib = ref.lib
        lib.dfsref_sample_prepare.restype = C.c_void_p
        lib.dfsref_sample_prepare.argtypes = [C.c_int64] * 6 + [C.c_double, C.c_int, C.c_int]
        lib.dfsref_sample_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
        lib.dfsref_sample_free.argtypes = [C.c_void_p]
        self.lib = lib
        self.ctx = lib.dfsref_sample_prepare(self.dims[0], self.dims[1], self.dims[2], self.d, self.B, self.Bs,
                                             self.gamma, self.heads_s, self.threads)

    def run(self, units_per_head):
        C = self.C
        sec, fixed = C.c_double(), C.c_double()
        if self.lib.dfsref_sample_run(self.ctx, units_per_head, self.threads, C.byref(sec), C.byref(fixed)):
            raise RuntimeError(self.ref._err().decode())
        units = self.heads_s * units_per_head
        call_s = fixed.value * math.ceil(self.H / self.threads) + sec.value * (self.H * self.m) / units
        return call_s, sec.value, fixed.value, units

    def describe(self, call_s, units_s, fixed_s, units, reps=1):
        return (f"reference dfs:: functions (oracle/_ref, unmodified sources) on {self.threads} host threads: "
                f"per-head reorder + key pooling {fixed_s:.2f}s for {self.heads_s} heads, then {units} of "
                f"{self.H * self.m} (head, query-block) units (pooled scoring + top-K + attend_row over "
                f"K={self.ref.topk_count(self.gamma, self.m)} blocks) in {units_s:.2f}s"
                + (f" (median of {reps})" if reps > 1 else "") +
                f"; extrapolated to one {self.H}-head call = {call_s:.0f}s")

    def close(self):
        if self.ctx:
            self.lib.dfsref_sample_free(self.ctx)
            self.ctx = None


def run_reference(args, wl):
    """Reference arm: the reference's own CPU implementation (oracle/_ref, built
    from /root/reference) on a bounded sample of the same call, all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    dims, H, d, B, Bs, gamma = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"], wl["gamma"]
    n = dims[0] * dims[1] * dims[2]
    dense_flops = 4.0 * d * n * n * H
    rs = RefSampler(wl)
    if rs.ctx is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdfsref.so not built (needs "
                          "/root/reference at build time)"}))
        return
    # each step samples ~units_per_thread (head, query-block) units per host thread; by default
    # sized so the whole --warmup + --steps run stays near 2.5 minutes (~0.6 s per unit per thread)
    upt = args.ref_units_per_thread
    if upt <= 0:
        upt = max(1, int(150.0 / max(1, args.warmup + args.steps) / 0.6))
    units_per_head = max(1, (rs.threads * upt) // rs.heads_s)
    runs = []
    for i in range(args.warmup + args.steps):
        r = rs.run(units_per_head)
        if i >= args.warmup:
            runs.append(r)
    rs.close()
    runs.sort(key=lambda r: r[0])
    call_s, units_s, fixed_s, units = runs[len(runs) // 2]
    value = dense_flops / call_s / 1e12
    sample = rs.describe(call_s, units_s, fixed_s, units, reps=len(runs))
    out = {"metric": metric_for(args.workload, wl), "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": call_s * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic iid normal (content does not change CPU op count)",
           "config": {"workload": wl["name"], "tokens": n, "heads": H, "d": d, "block": B, "sub_block": Bs,
                      "gamma": gamma},
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": rs.threads, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def cpu_baseline(wl, budget_s=20.0):
    """The same sample as the reference arm, sized to ~budget_s of CPU work (rank 0, N=1)."""
    rs = RefSampler(wl)
    if rs.ctx is None:
        return {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    # ~0.4 s of reference work per (head, query block) unit at HY on one core
    units_per_head = max(1, int(budget_s / 0.4) * rs.threads // rs.heads_s // 2)
    call_s, units_s, fixed_s, units = rs.run(units_per_head)
    rs.close()
    d, n, H = wl["d"], rs.n, wl["heads"]
    return {"value": 4.0 * d * n * n * H / call_s / 1e12, "unit": "TFLOP/s", "cores": rs.threads,
            "kind": "reference", "sample": rs.describe(call_s, units_s, fixed_s, units), "ms_per_call": call_s * 1e3}


TRAJ_BUDGETS = {"W4": (0.15,), "W7": (0.3, 0.2, 0.1), "HY": (0.3, 0.2, 0.1), "C": (0.2,)}


def run_trajectory_bench(args, wl, dfs, dev, world, rank, local, dist):
    """Config W4 / W7 of BASELINE.json: masks cached across a 50-step schedule
    (scheduler.hpp:22-28 defaults: warmup 25%, phase 25% per budget, Delta = 12)."""
    import torch

    dims, H, d, B, Bs = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"]
    n = dims[0] * dims[1] * dims[2]
    h0, h1 = rank * H // world, (rank + 1) * H // world
    q, k, v = smooth_fields(dims, h1 - h0, d, seed=1000 + rank, device=dev)
    budgets = TRAJ_BUDGETS.get(args.workload, (wl["gamma"],))
    T = 50
    sched = dfs.SparsitySchedule(total_steps=T, warmup_fraction=0.25, phase_budgets=budgets,
                                 phase_fraction=min(0.25, 0.75 / len(budgets)), update_interval=12)
    cache = dfs.MaskCache()
    params = dfs.ScoringParams(B, Bs)
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    kinds = {"dense": [], "update": [], "reuse": []}
    dense_flops_total = 0.0
    # warm-up: one whole trajectory (>= args.warmup steps), so the update steps' kernels
    # (pooling, scoring, top-K) and workspaces are warm too, then an empty mask cache
    for i in range(max(args.warmup, T)):
        dfs.run_step(q, k, v, dims, params, sched, cache, layer=0, step=i % T, out=out)
    barrier()
    cache.clear()
    steps = max(args.steps, T)
    with ClockSampler(local) as clocks:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(steps):
            s = i % T
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _, st = dfs.run_step(q, k, v, dims, params, sched, cache, layer=0, step=s, out=out)
            b.record(stream)
            kind = "dense" if st.dense else ("update" if any(st.mask_updated) else "reuse")
            kinds[kind].append((a, b))
            dense_flops_total += 4.0 * d * n * n * H
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1) / steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    per_kind = {kk: (statistics.mean(a.elapsed_time(b) for a, b in vv) if vv else None, len(vv))
                for kk, vv in kinds.items()}
    if rank != 0:
        dist.destroy_process_group()
        return
    res = {"metric": metric_for(args.workload, wl) + " (averaged over a 50-step mask-caching trajectory)",
           "value": dense_flops_total / steps / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
           "steps": steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "bf16", "data": "synthetic smooth Gaussian video fields",
           "config": {"workload": wl["name"], "schedule": {"total_steps": T, "warmup_fraction": 0.25,
                                                          "phase_budgets": list(budgets), "update_interval": 12},
                      "parallelism": f"head-shard x{world}"},
           "per_step_kind_ms": {kk: {"mean_ms": m_, "count": c_} for kk, (m_, c_) in per_kind.items()},
           "gpu_launches": None, "clocks": clocks.summary()}
    print(json.dumps(res))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="HY", choices=sorted(WORKLOADS))
    ap.add_argument("--gamma", type=float, default=None,
                    help="override the workload's block budget (W7 sparsity sweep: 0.30 ... 0.05)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-units-per-thread", type=int, default=0,
                    help="reference arm sample size per step (0: sized for a ~2.5 min run)")
    ap.add_argument("--profile", action="store_true", help="only run warmup+steps of the step (for ncu)")
    ap.add_argument("--trajectory", action="store_true",
                    help="diffusion trajectory: T=50 steps, 25%% dense warmup, phase budgets, mask update every "
                         "Delta=12 sparse steps (the device mask cache serves the other steps); reports per-step "
                         "averages over the whole schedule instead of the update-step call")
    ap.add_argument("--ulysses-nccl", action="store_true",
                    help="with --ulysses: exchange with torch.distributed NCCL all_to_all + pack/unpack copies "
                         "instead of the exchange fused into K2/K5 over peer memory (dfs_alltoall_run_step)")
    ap.add_argument("--ulysses", action="store_true",
                    help="sequence-sharded inputs [N/P, H, d]: NCCL all-to-all to heads, step, all-to-all back "
                         "(inside the timed region); default: head-sharded inputs, no collective")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.gamma is not None:
        wl["gamma"] = args.gamma
        wl["name"] = wl["name"].split(",")[0] + f", {round(100 * (1 - args.gamma))}% block sparsity (gamma={args.gamma})"
    if args.impl == "reference":
        run_reference(args, wl)
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` outside torchrun: launch the N ranks (one per GPU, NCCL)
        # exactly as the driver does, and pass their rank-0 line through
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))

    import torch
    import torch.distributed as dist

    import paper_2605_23445_b200 as dfs
    from paper_2605_23445_b200 import ops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DFS_BENCH_RANKS_PER_GPU > 1 (tests of the multi-rank code on one GPU) maps several
    # ranks to one device and uses gloo; the real runs are one rank per GPU over NCCL
    share = int(os.environ.get("DFS_BENCH_RANKS_PER_GPU", "1"))
    local = local // share
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share > 1:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    dims, H, d, B, Bs, gamma = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"], wl["gamma"]
    n = dims[0] * dims[1] * dims[2]
    m = -(-n // B)
    h0, h1 = rank * H // world, (rank + 1) * H // world
    hl = h1 - h0
    if args.trajectory:
        return run_trajectory_bench(args, wl, dfs, dev, world, rank, local, dist)
    ulysses_mode = args.ulysses and world > 1
    if ulysses_mode:
        from paper_2605_23445_b200 import ulysses

        if n % world or H % world:
            raise SystemExit(f"--ulysses needs tokens and heads divisible by {world}")
        nl = n // world
        full = smooth_fields(dims, H, d, seed=1000, device=dev)  # same field on every rank; keep my token shard
        ql, kl, vl = (x[rank * nl:(rank + 1) * nl].contiguous() for x in full)
        del full
        q, k, v = ulysses.seq_to_head([ql, kl, vl])  # head-local view, for the kernel breakdown only
        ol = torch.empty_like(ql)
        exch = None if args.ulysses_nccl else ulysses.PeerExchange(ql, kl, vl, ol)
    else:
        q, k, v = smooth_fields(dims, hl, d, seed=1000 + rank, device=dev)
    params = dfs.ScoringParams(B, Bs)
    sched = dfs.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(gamma,), phase_fraction=1.0,
                                 update_interval=1)
    cache = dfs.MaskCache()
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        if ulysses_mode and exch is not None:
            exch.fused_run_step(dims, params, sched, cache, layer=0, step=0)
        elif ulysses_mode:
            ulysses.ulysses_run_step(ql, kl, vl, dims, params, sched, cache, layer=0, step=0)
        else:
            dfs.run_step(q, k, v, dims, params, sched, cache, layer=0, step=0, out=out)

    for _ in range(args.warmup):
        step()
    barrier()
    if args.profile:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        return

    # ---- timed region: K full update-step calls --------------------------------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # ---- the same call under CUPTI (torch.profiler, after the timed region): per-kernel
    # durations inside the update-step call, grouped by stage (the CUDA-event decomposition
    # below times each stage alone, so its clocks can differ from the step's)
    step_kernels = None
    if not ulysses_mode:
        try:
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                for _ in range(3):
                    step()
                torch.cuda.synchronize()
            stages = {"K2_permute_pool": ("permute_kernel", "Memset"), "K3_score": ("absmax", "split_kernel", "score_"),
                      "K4_topk": ("topk", "lut_ptr"), "K5_attn": ("attn_",)}
            acc = {k: 0.0 for k in stages}
            acc["other"] = 0.0
            evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
            for e in evs:
                dur = (e.time_range.end - e.time_range.start) / 1e3 / 3
                key = next((k for k, pats in stages.items() if any(pt in e.name for pt in pats)), "other")
                acc[key] += dur
            span = (max(e.time_range.end for e in evs) - min(e.time_range.start for e in evs)) / 1e3 / 3
            step_kernels = {k: round(v, 4) for k, v in acc.items()}
            step_kernels["span_per_call"] = round(span, 4)
            step_kernels["how"] = ("3 calls under torch.profiler (CUPTI) right after the timed region: kernel "
                                   "durations per call by stage; a 50 ms burst runs at a higher clock than the "
                                   "power-capped timed loop")
        except Exception as ex:  # pragma: no cover
            step_kernels = {"failed": str(ex)}

    # ---- decomposition (per-kernel CUDA-event timing on the launching stream) ---
    # the same kernels run_step launches: K2 read-only pooling of q and k in Hilbert order,
    # K3, K4, and K5 gathering the Hilbert-ordered rows itself (fused reorder + unpermute)
    perm = dfs.hilbert3d_order(dims)
    pq = ops.pool_gathered(q, perm, Bs)
    kh, pk = ops.permute_to_hnd(k, perm, Bs)
    vh, _ = ops.permute_to_hnd(v, perm, 0)
    S = ops.score_pooled(pq, pk, n, params)
    lut = dfs.topk_lut(S, gamma)
    K = lut.shape[-1]
    ptr = ops.lut_row_ptr(hl, m, K, device=dev)
    o2 = torch.empty_like(q)

    def timed(fn, reps=5):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    t_perm = timed(lambda: (ops.pool_gathered(q, perm, Bs), ops.permute_to_hnd(k, perm, Bs),
                            ops.permute_to_hnd(v, perm, 0)))
    t_score = timed(lambda: ops.score_pooled(pq, pk, n, params, out=S))
    t_topk = timed(lambda: dfs.topk_lut(S, gamma))
    t_attn = timed(lambda: dfs.sparse_attention_csr(q, kh, vh, ptr, lut.reshape(-1), B, layout=1, out_layout=0,
                                                    in_rows=perm.forward, out_rows=perm.forward, out=o2))
    # reuse-step call: mask from the cache, no scoring
    sched_reuse = dfs.SparsitySchedule(total_steps=2, warmup_fraction=0.0, phase_budgets=(gamma,),
                                       phase_fraction=1.0, update_interval=2)
    dfs.run_step(q, k, v, dims, params, sched_reuse, cache, layer=1, step=0, out=out)
    t_reuse = timed(lambda: dfs.run_step(q, k, v, dims, params, sched_reuse, cache, layer=1, step=1, out=out))
    # K1 (token order): once per lattice geometry, cached by the handle, so outside the call
    t_k1 = timed(lambda: dfs.hilbert3d_order(dims))
    # LUT overlap of query-block pairs (2u, 2u+1): |I_u ∪ I_u+1| / K, and the
    # fraction of query blocks that select their own (diagonal) block
    pairs = lut[:, : (m // 2) * 2].reshape(hl, m // 2, 2 * K)
    srt = pairs.sort(-1).values
    union = 1 + (srt[..., 1:] != srt[..., :-1]).sum(-1)
    diag = (lut == torch.arange(m, device=dev).view(1, m, 1)).any(-1).float().mean().item()
    overlap = {"pair_union_over_K_mean": float(union.float().mean().item() / K),
               "pair_union_over_K_min": float(union.min().item() / K),
               "pair_union_over_K_max": float(union.max().item() / K), "diag_selected_frac": diag}

    exec_flops = executed_flops(lut, n, B, d)
    if world > 1:
        ef = torch.tensor([exec_flops], device=dev, dtype=torch.float64)
        dist.all_reduce(ef)
        exec_flops = float(ef.item())
    dense_flops = 4.0 * d * n * n * H
    peak_burst, peak_sus, hbm, peak_kind = peaks()
    attn_flops_local = executed_flops(lut, n, B, d)
    achieved = attn_flops_local / (t_attn * 1e-3) / 1e12

    # ---- e2e: host buffers through the public API, copies inside the timed region.
    # Every step copies its own inputs host->device (pinned) and its output back;
    # two buffer sets and separate copy streams let step i+1's upload and step
    # i-1's download overlap step i's kernels (PCIe is the bound, not the GPU).
    e2e = None
    src = (ql, kl, vl) if ulysses_mode else (q, k, v)
    host_in = [tuple(x.cpu().pin_memory() for x in src) for _ in range(2)]
    host_out = [torch.empty(src[0].shape, dtype=src[0].dtype).pin_memory() for _ in range(2)]
    dev_in = [tuple(torch.empty_like(x) for x in src) for _ in range(2)]
    dev_out = [torch.empty_like(src[0]) for _ in range(2)]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def upload(i):
        b = i % 2
        with torch.cuda.stream(h2d_s):
            h2d_s.wait_event(ev_done[b])  # step i-2 finished reading these device inputs
            for x_d, x_h in zip(dev_in[b], host_in[b]):
                x_d.copy_(x_h, non_blocking=True)
            ev_in[b].record(h2d_s)

    def e2e_step(i):
        # step i's upload was enqueued one step ahead (before step i-1's run_step, whose
        # non-finite read-back blocks the host until that step's K2 has run): the copy
        # engine streams uploads back to back instead of idling for a K2 per call
        b = i % 2
        stream.wait_event(ev_in[b])
        stream.wait_event(ev_out[b])  # step i-2's output has left the device buffer
        qd, kd, vd = dev_in[b]
        if ulysses_mode and exch is not None:  # shards registered once: stage through them
            for x_s, x_d in zip((ql, kl, vl), (qd, kd, vd)):
                x_s.copy_(x_d)
            exch.fused_run_step(dims, params, sched, cache, layer=0, step=0)
            dev_out[b].copy_(ol)
        elif ulysses_mode:
            dev_out[b].copy_(ulysses.ulysses_run_step(qd, kd, vd, dims, params, sched, cache, layer=0, step=0)[0])
        else:
            dfs.run_step(qd, kd, vd, dims, params, sched, cache, layer=0, step=0, out=dev_out[b])
        ev_done[b].record(stream)
        with torch.cuda.stream(d2h_s):
            d2h_s.wait_event(ev_done[b])
            host_out[b].copy_(dev_out[b], non_blocking=True)
            ev_out[b].record(d2h_s)

    upload(0)
    for i in range(2):
        if i + 1 < 2:
            upload(i + 1)
        e2e_step(i)
    barrier()
    n_e2e = max(4, args.steps)
    a = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    h2d_s.wait_event(a)  # every timed upload starts inside the timed region
    upload(0)
    for i in range(n_e2e):
        if i + 1 < n_e2e:
            upload(i + 1)
        e2e_step(i)
    d2h_s.synchronize()
    end = torch.cuda.Event(enable_timing=True)
    stream.wait_stream(d2h_s)
    end.record(stream)
    barrier()
    e2e_ms = a.elapsed_time(end) / n_e2e
    et = torch.tensor([e2e_ms], device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_ms = float(et.item())
    h2d = sum(x.numel() * x.element_size() for x in src) * world
    d2h = src[0].numel() * src[0].element_size() * world
    e2e = {"value": dense_flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_call": e2e_ms,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "how": "public API dfs.run_step" + ((" under ulysses_run_step (NCCL)" if args.ulysses_nccl else
                                                 " under PeerExchange.fused_run_step") if ulysses_mode else "") +
                  " on device copies of pinned host inputs, output read back every step; each step's upload is "
                  "enqueued one step ahead on its own copy stream and downloads run on another, so copies of "
                  "neighbouring steps overlap the kernels"}

    if rank != 0:
        dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(wl)
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "sample": f"failed: {ex}"}
    # our kernels per update-step call (dfs_run_step; tools/step_timeline.py lists them): q pooling
    # (read-only, gathered), k permute+pool, v permute, scorer prep (q+k absmax, q+k fp16 split with
    # the logit factor) + 1 tcgen05 scorer, 1 top-K, 1 LUT row pointers, 1 attention (TMA-gathered Q
    # reorder + fused unpermute)
    launches_per_step = 3 + 3 + 1 + 1 + 1
    res = {
        "metric": metric_for(args.workload, wl), "value": dense_flops / (ms_max * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic smooth Gaussian video fields (4 smoothing rounds), generated on device",
        "config": {"workload": wl["name"], "tokens": n, "heads": H, "heads_per_gpu": hl, "d": d, "block": B,
                   "sub_block": Bs, "gamma": gamma, "K": K, "M": m, "parallelism": ((f"ulysses NCCL all-to-all x{world}" if args.ulysses_nccl else
                                    f"ulysses all-to-all fused into K2/K5 (P2P) x{world}") if ulysses_mode
                                   else f"head-shard x{world}"),
                   "l2": (f"q/k/v/o {n * hl * d * 2 / 1e6:.0f} MB bf16 each, {4 * n * hl * d * 2 / 1e6:.0f} MB touched "
                          f"per step + the permuted K/V copies > 126 MB L2 (no flush between steps)")},
        "ms_per_call_mask_reuse": t_reuse,
        "order_K1_ms_per_geometry": t_k1,
        "lut_overlap": overlap,
        "executed_tflop_per_call": exec_flops / 1e12, "dense_equiv_tflop_per_call": dense_flops / 1e12,
        "executed_tflops": exec_flops / (ms_max * 1e-3) / 1e12,
        "step_kernel_ms_cupti": step_kernels,
        "breakdown_ms": {"reorder_pool_K2": t_perm, "score_K3": t_score, "topk_K4": t_topk,
                         "attn_unpermute_K5": t_attn},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"kernel": "K5 block-sparse attention (TMA-gathered Q reorder + fused unpermute)", "bound": "tensor",
                     "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s", "frac": achieved / peak_burst,
                     "peak_kind": f"{peak_kind} bf16 burst", "traffic": k5_traffic(args.workload, hl),
                     "traffic_unit": "DRAM bytes per launch (ncu, read+write)",
                     "algorithmic_bytes": 4.0 * n * hl * d * 2,
                     "peak_sustained": peak_sus, "frac_sustained": achieved / peak_sus,
                     "algorithmic": "executed FLOPs 4*d*sum(r_u*c_v) per launch / CUDA-event duration"},
        "path_fraction_of_peak": exec_flops / (ms_max * 1e-3) / 1e12 / peak_burst,
        "path_fraction_of_sustained_peak": exec_flops / (ms_max * 1e-3) / 1e12 / peak_sus,
        "e2e": e2e,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(res))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

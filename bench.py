#!/usr/bin/env python3
"""Benchmark: padding-free FP8 grouped GEMM on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[1], the residual sweep): 8 experts,
per-expert B [8, 7168, 4096] e4m3 with 128x128 fp32 scales, N=4096, K=7168.
For each r in 1..127 the groups are M_g = 128*g + r, g = 0..7, so every
M_g mod 128 occurs and all 7 residual store heights are exercised.  One bench
"step" is a pass over all 127 problems (127 kernel launches).  ``value`` is
valid TFLOP/s = sum 2*M_g*N*K / time.  It is whole-job over all ranks.  Each
rank owns its own 8 experts (expert parallel, no data-path collective), so
scaling is weak.

Also reported, all on the same GPU and in the same run:
* the pad-to-128 + padded-GEMM baseline (K2 pad kernel + the same GEMM on
  128-aligned groups + K3 unpad): its TFLOP/s, the speedup and the memory saved;
* ``e2e``: the same metric through the public API with host buffers.  Per step
  it copies the A rows, A scales and group sizes H2D from pinned memory and
  copies every problem's C back D2H.  Expert weights stay resident, as model
  parameters do;
* ``roofline``: the GEMM kernel's achieved TFLOP/s per launch (CUDA events on
  the launch stream) against the FP8 dense peak (2 x the measured bf16 peak);
* ``cpu_baseline``: the CPU oracle (a C port of the reference's run_adaptive,
  oracle/) on a bounded sample of the same workload, using every host core;
* ``extra``: the other BASELINE.json configs (DeepSeek-V3 gate+up and down,
  Qwen3-235B forward + dgrad), each with its padded-baseline speedup.

``--impl reference`` times the reference's CPU implementation of the path
(the oracle port; the reference itself is numpy-only Python) on the same
metric and config.  Rank 0 alone runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "valid TFLOPS & speedup vs pad+padded FP8 grouped GEMM; % FP8 peak; memory saved"
UNIT = "TFLOP/s"
FP8_SPEC_TFLOPS = 4500.0


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- workloads
def sweep_problems():
    """configs[1]: r = 1..127, M_g = 128*g + r for g = 0..7."""
    return [tuple(128 * g + r for g in range(8)) for r in range(1, 128)]


def deepseek_gateup_sizes(seed=0, tokens=32768, topk=8, experts=256, local=32, zipf=0.8):
    """Zipf-skewed top-8 routing of T tokens over 256 experts (seeded Gumbel
    top-k); the local experts of EP rank 0 of 8 (a seeded random subset)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    perm = rng.permutation(experts)
    logp = -zipf * np.log(np.arange(1, experts + 1, dtype=np.float64))[np.argsort(perm)]
    counts = np.zeros(experts, dtype=np.int64)
    for lo in range(0, tokens, 4096):
        n = min(4096, tokens - lo)
        g = rng.gumbel(size=(n, experts)) + logp[None, :]
        top = np.argpartition(-g, topk, axis=1)[:, :topk]
        counts += np.bincount(top.ravel(), minlength=experts)
    return counts, counts[:local]


def headline_operands(seed, m_alloc, n=4096, k=7168, experts=8):
    """The headline's resident operands as numpy arrays, drawn from one seed, so the GPU arm
    and the reference (CPU) arm compute on the very same bytes: uniform finite e4m3 codes
    (no NaN code) and positive fp32 scales 2^[-12,-5) x [0.5, 1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    kb, nb = -(-k // 128), -(-n // 128)

    def codes(shape):
        c = rng.integers(0, 256, size=shape, dtype=np.uint8)
        c[(c & 0x7F) == 0x7F] -= 1
        return c

    def scales(shape):
        e = rng.integers(-12, -4, size=shape).astype(np.float32)
        return ((rng.random(shape, dtype=np.float32) * np.float32(0.5) + np.float32(0.5)) * np.exp2(e)).astype(
            np.float32)

    return codes((m_alloc, k)), scales((m_alloc, kb)), codes((experts, k, n)), scales((experts, kb, nb))


HEADLINE_SEED = 1000  # + rank: each rank owns its own experts
SAMPLE_R = 64         # the CPU sample / self-check problem of the sweep: M_g = 128 g + 64


def headline_config(world, exact):
    """The headline's config dict; both arms print exactly this."""
    return {
        "workload": "residual sweep (BASELINE.json configs[1]): per rank 8 experts, M_g=128g+r, r=1..127 "
                    "(127 grouped GEMMs per step), N=4096, K=7168, per-expert B [8,7168,4096]",
        "N": 4096, "K": 7168, "groups": 8, "rows_per_step": sum(sum(s) for s in sweep_problems()),
        "parallelism": f"ep{world} (experts sharded, no data-path collective)",
        "l2": "inputs > L2: B is 235 MB per rank (126 MB L2), re-read from HBM every launch; no flush",
        "promotion": "exact fmul+fadd" if exact else "ffma2",
        "operands": f"bench.headline_operands(seed={HEADLINE_SEED}+rank): identical bytes in both arms",
    }


def _codes(torch, shape, gen, device):
    c = torch.randint(0, 256, shape, dtype=torch.uint8, device=device, generator=gen)
    return torch.where((c & 0x7F) == 0x7F, c - 1, c)  # never a NaN code


def _scales(torch, shape, gen, device):
    e = torch.randint(-12, -4, shape, device=device, generator=gen).float()
    return (torch.rand(shape, device=device, generator=gen) * 0.5 + 0.5) * torch.exp2(e)


class Problem:
    """Resident device operands for one weight set and a list of group-size vectors."""

    def __init__(self, torch, name, sizes_list, n, k, experts, device, seed, b_layout="kn", host=None):
        self.name, self.n, self.k, self.G = name, n, k, experts
        self.sizes_list = [tuple(int(x) for x in s) for s in sizes_list]
        self.m_alloc = max(sum(s) for s in self.sizes_list)
        kb, nb = -(-k // 128), -(-n // 128)
        if host is not None:  # numpy operands (headline_operands), uploaded once
            self.a, self.sa, self.b, self.sb = (torch.from_numpy(x).to(device) for x in host)
        else:
            gen = torch.Generator(device=device).manual_seed(seed)
            self.a = _codes(torch, (self.m_alloc, k), gen, device)
            self.sa = _scales(torch, (self.m_alloc, kb), gen, device)
            if b_layout == "kn":
                self.b = _codes(torch, (experts, k, n), gen, device)
                self.sb = _scales(torch, (experts, kb, nb), gen, device)
            else:
                self.b = _codes(torch, (experts, n, k), gen, device)
                self.sb = _scales(torch, (experts, nb, kb), gen, device)
        self.b_layout = b_layout
        self.gs = [torch.tensor(s, dtype=torch.int32, device=device) for s in self.sizes_list]
        self.out = torch.empty((self.m_alloc, n), dtype=torch.bfloat16, device=device)
        self.flops = [2.0 * sum(s) * n * k for s in self.sizes_list]

    def algorithmic_bytes(self, sizes):
        """every operand touched once, no padding."""
        n, k = self.n, self.k
        kb, nb = -(-k // 128), -(-n // 128)
        active = sum(1 for s in sizes if s > 0)
        return sum(sizes) * (k + 4 * kb + 2 * n) + active * (n * k + 4 * kb * nb)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits", "-lms", "100"],
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        try:
            while not self._stop.is_set():
                line = p.stdout.readline()
                if not line:
                    break
                self.rows.append([x.strip() for x in line.split(",")])
        finally:
            p.terminate()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=2)

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        under = [x for x in sm if x > 500] or sm
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(under), "sm_max_mhz": float(self.rows[0][1]),
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- timing helpers
def _free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _timed_steps(torch, dist, world, step_fn, steps, warmup):
    for _ in range(warmup):
        step_fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step_fn()
    e.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = s.elapsed_time(e)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def _per_launch_ms(torch, launches, reps=3):
    """Average device duration of each launch, CUDA events on the launch stream."""
    stream = torch.cuda.current_stream()
    out = []
    for fn in launches:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in evs:
            a.record(stream)
            fn()
            b.record(stream)
        out.append(evs)
    torch.cuda.synchronize()
    return [sum(a.elapsed_time(b) for a, b in evs) / reps for evs in out]


def _flush_l2(torch, buf):
    buf.add_(1)


# ----------------------------------------------------------------------------- CPU baseline
def _parity(got_bits, want_bits):
    """tests/helpers.REL_TOL: |c - c_ref| <= 2^-7 max(|c_ref|, 2^-10 rowabsmax(c_ref)) per element."""
    got = (got_bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    ref = (want_bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    rowmax = np.abs(ref).max(axis=1, keepdims=True)
    bad = np.abs(got - ref) > 2.0 ** -7 * np.maximum(np.abs(ref), 2.0 ** -10 * rowmax)
    return {"out_of_tol": int(bad.sum()), "bit_identical": float((got_bits == want_bits).mean()),
            "elements": int(ref.size)}


def cpu_sample(threads, ops, target_s=10.0, got_bits=None):
    """Time the CPU oracle (C port of the reference's run_adaptive semantics, every host
    thread) on a bounded sample of the headline: the r=SAMPLE_R problem of the sweep
    (M_g = 128 g + 64, 8 experts, K=7168) over the headline's own operands ``ops``
    (headline_operands), on a 128-aligned column slice calibrated to ~target_s seconds.
    With ``got_bits`` (the GPU arm's C of that problem, uint16 [m, 4096]) the sample is
    also the parity check of the bench's own output: out-of-tolerance count and the
    bit-identical fraction on the sampled columns."""
    from oracle import oracle as orc

    ac, asc, bc, bsc = ops
    sizes = tuple(128 * g + SAMPLE_R for g in range(8))
    n, k = bc.shape[-1], bc.shape[-2]
    m = sum(sizes)
    ac, asc = ac[:m], asc[:m]
    out = np.zeros((m, n), dtype=np.uint16)
    orc.grouped_gemm(ac, asc, bc, bsc, sizes, n_range=(0, 128), threads=threads, out=out)  # warm pages
    t0 = time.perf_counter()
    orc.grouped_gemm(ac, asc, bc, bsc, sizes, n_range=(0, 256), threads=threads, out=out)
    per_col = (time.perf_counter() - t0) / 256
    cols = int(min(n, max(128, int(target_s / max(per_col, 1e-9)) // 128 * 128)))
    t0 = time.perf_counter()
    orc.grouped_gemm(ac, asc, bc, bsc, sizes, n_range=(0, cols), threads=threads, out=out)
    dt = time.perf_counter() - t0
    flops = 2.0 * m * cols * k
    sample = (f"residual sweep r={SAMPLE_R} (M_g=128g+{SAMPLE_R}, 8 experts, K=7168) on the headline's operands, "
              f"N-slice [0,{cols}) of {n}: {flops:.3e} FLOP in {dt:.2f}s")
    par = None if got_bits is None else _parity(got_bits[:m, :cols], out[:, :cols])
    return flops / dt / 1e12, dt, sample, par


def reference_arm(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path (oracle port, all
    host threads) on the same metric, config and operands as the GPU arm, rank 0 only."""
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    from oracle import oracle as orc  # noqa: F401  (built by __graft_entry__.build)

    ops = headline_operands(HEADLINE_SEED, max(sum(s) for s in sweep_problems()))
    vals = []
    sample = ""
    # each step is a bounded sample of the headline workload (~5 s)
    for i in range(args.warmup + args.steps):
        v, dt, sample, _ = cpu_sample(threads, ops, target_s=5.0 if i >= args.warmup else 1.0)
        if i >= args.warmup:
            vals.append((v, dt))
    value = statistics.median(v for v, _ in vals)
    ms = statistics.median(dt for _, dt in vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp8_e4m3 (fp32 accumulate, bf16 out)",
        "data": "synthetic (uniform finite e4m3 codes, positive fp32 scales; per-rank expert weights)",
        "config": headline_config(world, args.exact),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- main arm
def run_problem_set(torch, tg, prob, iters, warmup, flush=None, exact=False):
    """Time adaptive vs pad+padded on every size vector of ``prob``."""
    ws = tg.PaddedWorkspace(prob.m_alloc, prob.G, prob.k, prob.n, prob.a.device)
    outs = prob.out

    def adaptive():
        for gs in prob.gs:
            tg.grouped_gemm_fp8(prob.a, prob.sa, prob.b, prob.sb, gs, b_layout=prob.b_layout, out=outs,
                                exact_promotion=exact, pdl_overlap=True)

    def padded(unpad=True):
        for gs in prob.gs:
            tg.padded_grouped_gemm_fp8(prob.a, prob.sa, prob.b, prob.sb, gs, ws, b_layout=prob.b_layout, out=outs,
                                       unpad=unpad, exact_promotion=exact)

    # three rounds in rotating order, median per arm: the first block after an idle gap runs at
    # a higher clock (power state), so a fixed order would favour whichever arm goes first
    arms = [("adaptive", adaptive), ("padded", padded), ("padded_no_unpad", lambda: padded(False))]
    times = {name: [] for name, _ in arms}
    for rnd in range(3):
        for name, fn in arms[rnd:] + arms[:rnd]:
            for _ in range(warmup):
                fn()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(iters):
                fn()
            e.record()
            torch.cuda.synchronize()
            times[name].append(s.elapsed_time(e) / iters)
    res = {name: sorted(v)[1] for name, v in times.items()}
    flops = sum(prob.flops)
    return {k: flops / (v * 1e-3) / 1e12 for k, v in res.items()}, res, ws.nbytes()


def per_residue_speedups(torch, tg, prob, iters=3):
    """Speedup over pad + padded for EVERY residue r of the sweep (the north star's "beats
    pad+padded across the residual sweep"): each size vector timed alone, both paths, with and
    without the unpad copy.  Back-to-back launches of one size vector (events around them)."""
    ws = tg.PaddedWorkspace(prob.m_alloc, prob.G, prob.k, prob.n, prob.a.device)

    def timed(fn):
        fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / iters

    sp, sp_nu = [], []
    for gs in prob.gs:
        t_a = timed(lambda: tg.grouped_gemm_fp8(prob.a, prob.sa, prob.b, prob.sb, gs, out=prob.out))
        t_p = timed(lambda: tg.padded_grouped_gemm_fp8(prob.a, prob.sa, prob.b, prob.sb, gs, ws, out=prob.out))
        t_n = timed(lambda: tg.padded_grouped_gemm_fp8(prob.a, prob.sa, prob.b, prob.sb, gs, ws, out=prob.out,
                                                       unpad=False))
        sp.append(t_p / t_a)
        sp_nu.append(t_n / t_a)
    worst = min(range(len(sp)), key=lambda i: sp_nu[i])
    return {"min": min(sp), "max": max(sp), "min_no_unpad": min(sp_nu), "max_no_unpad": max(sp_nu),
            "r_of_min_no_unpad": worst + 1, "all_above_1": bool(min(sp_nu) > 1.0),
            "per_r_no_unpad": [round(x, 3) for x in sp_nu]}


def measured_peak_deltas(torch, tg, prob, sizes):
    """the allocator's peak-memory delta of one call of each path (outputs,
    workspace and all), on the largest size vector of the sweep."""
    gs = torch.tensor(sizes, dtype=torch.int32, device=prob.a.device)
    out = {}
    for name in ("padding_free", "padded"):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        if name == "padding_free":
            c = tg.grouped_gemm_fp8(prob.a[:sum(sizes)], prob.sa[:sum(sizes)], prob.b, prob.sb, gs)
        else:
            ws = tg.PaddedWorkspace(sum(sizes), prob.G, prob.k, prob.n, prob.a.device)
            c = tg.padded_grouped_gemm_fp8(prob.a[:sum(sizes)], prob.sa[:sum(sizes)], prob.b, prob.sb, gs, ws)
        torch.cuda.synchronize()
        out[name + "_peak_delta_bytes"] = int(torch.cuda.max_memory_allocated() - base)
        del c
        if name == "padded":
            del ws
    out["sizes"] = list(sizes)
    return out


def _spawn(argv, gpus):
    """--gpus N without a torchrun environment: run this script again under
    torch.distributed.run, one rank per GPU (127.0.0.1 rendezvous), and return its status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve())] + argv
    return subprocess.call(cmd)


def dry_run(args, rank, world):
    """--dry-run: the multi-rank plumbing without a GPU (gloo): rank setup, the barrier-bracketed
    timed region, the max over ranks and rank 0's single JSON line.  The step is a fixed
    host workload, so the line carries no GEMM number ("dry_run": true)."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    x = np.random.default_rng(rank).standard_normal((256, 256)).astype(np.float32)
    for _ in range(args.warmup):
        x @ x
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x @ x
    ms = (time.perf_counter() - t0) * 1e3
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    if rank == 0:
        flops = world * args.steps * 2.0 * 256 ** 3
        print(json.dumps({"metric": METRIC, "value": flops / (ms * 1e-3) / 1e12, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dry_run": True,
                          "config": headline_config(world, args.exact)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--exact", action="store_true", help="two-rounding promotion (TAGG_FLAG_EXACT_PROMOTION)")
    ap.add_argument("--ep1", action="store_true",
                    help="also run the DeepSeek-V3 down EP config (sequential vs overlapped) at one GPU")
    ap.add_argument("--profile-once", action="store_true", help="one step only (for ncu launch lists)")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing on CPU (gloo), no GPU work")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn(sys.argv[1:], args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        dry_run(args, rank, world)
        return
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2508_16584_b200 as tg

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    peaks, peaks_src = _peaks()
    fp8_peak = 2.0 * float(peaks["bf16_tflops"])

    # ---------------------------------------------------------------- headline: residual sweep
    probs = sweep_problems()
    ops = headline_operands(HEADLINE_SEED + rank, max(sum(s) for s in probs))
    P = Problem(torch, "residual_sweep", probs, 4096, 7168, 8, dev, seed=HEADLINE_SEED + rank, host=ops)
    flops_step = sum(P.flops)
    launches_per_step = len(probs)

    def make_step(exact):
        def step():
            # 127 independent GEMMs over resident operands: no launch writes the next one's
            # inputs, so each may overlap its predecessor's tail (TAGG_FLAG_PDL_OVERLAP)
            for gs in P.gs:
                tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out, exact_promotion=exact, pdl_overlap=True)
        return step

    step = make_step(args.exact)
    if args.profile_once:
        step()
        torch.cuda.synchronize()
        return

    def graph_of(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        return graph

    # The timed step is the 127 launches captured once as a CUDA graph and replayed (the same
    # kernels, arguments and programmatic-dependent-launch edges, without the host's per-launch
    # cost between them); the same launches issued one by one from the host are timed beside it
    # (value_eager).
    g_main = graph_of(step)
    with ClockSampler(local) as clk:  # sampled over warm-up + timed steps (100 ms period)
        ms_total = _timed_steps(torch, dist, world, g_main.replay, args.steps, args.warmup)
    clocks = clk.summary()
    ms_step = ms_total / args.steps
    value = world * flops_step / (ms_step * 1e-3) / 1e12
    half = max(2, args.steps // 2)
    # launch method alone: eager and graph blocks of equal length, alternated (E G E G) right
    # after the headline, so neither gets the faster first block after an idle gap (the power
    # state, not the launch method, made a single eager block after the graph look faster)
    blocks = {"eager": [], "graph": []}
    for name in ("eager", "graph", "graph", "eager", "eager", "graph"):
        fn = step if name == "eager" else g_main.replay
        blocks[name].append(_timed_steps(torch, dist, world, fn, half, 1) / half)
    ms_eager = sorted(blocks["eager"])[1]  # medians of three
    ms_graph_alt = sorted(blocks["graph"])[1]
    del g_main
    # the reference's own rounding order (engine.py:161-164: fl(acc + fl(inner * s))) timed as well
    g_other = graph_of(make_step(not args.exact))
    ms_other = _timed_steps(torch, dist, world, g_other.replay, half, 1) / half
    del g_other

    # ---------------------------------------------------------------- roofline (dominant kernel = the GEMM)
    launch_fns = [(lambda gs=gs: tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out,
                                                     exact_promotion=args.exact, pdl_overlap=True)) for gs in P.gs]
    per_launch = _per_launch_ms(torch, launch_fns)
    achieved = sum(P.flops) / (sum(per_launch) * 1e-3) / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "traffic_residual_sweep.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
    alg_bytes = sum(P.algorithmic_bytes(s) for s in P.sizes_list) / len(P.sizes_list)

    # ---------------------------------------------------------------- padded baseline, same GPU
    base_tf, base_ms, ws_bytes = run_problem_set(torch, tg, P, iters=half, warmup=1, exact=args.exact)
    mem_measured = measured_peak_deltas(torch, tg, P, P.sizes_list[0])
    per_r = per_residue_speedups(torch, tg, P)
    acc = [tg.account(s, 4096, 7168) for s in P.sizes_list]
    saved_pct = 100.0 * (1 - sum(a.bytes_actual for a in acc) / sum(a.bytes_padded for a in acc))

    # ---------------------------------------------------------------- e2e through the public API
    # Every one of the 127 problems is an independent host-buffer call: its own A rows, A scales
    # and group sizes H2D from pinned memory, its C rows D2H; expert weights stay resident, as
    # model parameters do.  hostpipe overlaps problem i's D2H and i+1's H2D with the GEMMs.
    from paper_2508_16584_b200.hostpipe import HostBatch, run_host_batches

    pin_a = P.a.cpu().pin_memory()
    pin_sa = P.sa.cpu().pin_memory()
    pin_gs = [g.cpu().pin_memory() for g in P.gs]
    host_c = torch.empty((P.m_alloc, P.n), dtype=torch.bfloat16).pin_memory()
    rows = [sum(s) for s in P.sizes_list]
    batches = [HostBatch(pin_a[:m], pin_sa[:m], gh, host_c) for m, gh in zip(rows, pin_gs)]
    h2d = sum(m * (P.k + 4 * (P.k // 128)) + g.numel() * 4 for m, g in zip(rows, pin_gs))
    d2h = sum(m * P.n * 2 for m in rows)

    def e2e_step():
        run_host_batches(batches, P.b, P.sb, exact_promotion=args.exact)

    e2e_ms = _timed_steps(torch, dist, world, e2e_step, half, 1) / half
    e2e_val = world * flops_step / (e2e_ms * 1e-3) / 1e12
    # the host link bounds it: PCIe is full duplex, so the larger direction sets the time
    e2e_link_gbs = max(h2d, d2h) / (e2e_ms * 1e-3) / 1e9

    # ---------------------------------------------------------------- CPU baseline + self-check (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sizes = tuple(128 * g + SAMPLE_R for g in range(8))
        c_chk = torch.empty((sum(sizes), P.n), dtype=torch.bfloat16, device=dev)
        tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, torch.tensor(sizes, dtype=torch.int32, device=dev), out=c_chk,
                            exact_promotion=args.exact)
        got = c_chk.view(torch.int16).cpu().numpy().view(np.uint16)
        threads = len(os.sched_getaffinity(0))
        v, dt, sample, par = cpu_sample(threads, ops, target_s=10.0, got_bits=got)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
               "parity_vs_gpu_output": dict(par, tolerance="|c-c_ref| <= 2^-7 max(|c_ref|, 2^-10 rowabsmax)",
                                            what=f"this run's GPU C of the r={SAMPLE_R} problem vs the CPU "
                                                 "oracle on the same operands and columns")}

    # ---------------------------------------------------------------- other BASELINE configs
    # secondary lines never cost the headline: a failure is recorded, not raised
    extra = {}
    if not args.no_extra:
        try:
            extra = run_extra(torch, tg, dev, rank, fp8_peak, args.exact)
        except Exception as exc:  # noqa: BLE001
            extra = {"error": f"{type(exc).__name__}: {exc}"}
    if world == 1 and args.ep1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    if world > 1 or args.ep1:
        try:
            extra["deepseek_v3_down_ep"] = run_ep_down(torch, dist, tg, dev, rank, world, fp8_peak, args.exact)
        except Exception as exc:  # noqa: BLE001
            extra["deepseek_v3_down_ep"] = {"error": f"{type(exc).__name__}: {exc}"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cfg = headline_config(world, args.exact)  # identical to the reference arm's config
    other = "value_ffma2" if args.exact else "value_exact"
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp8_e4m3 (fp32 accumulate, bf16 out)",
        "data": "synthetic (uniform finite e4m3 codes, positive fp32 scales; per-rank expert weights)",
        "config": cfg,
        "timing": ("timed step = one CUDA-graph replay of the 127 launches (captured once over the resident "
                   "operands; programmatic dependent launch chains them); value_eager: the same launches issued "
                   "one by one from the host, timed in blocks alternating with graph blocks after the headline "
                   "(value_graph_alternated: the graph blocks), E G G E E G; median block of each"),
        "value_eager": world * flops_step / (ms_eager * 1e-3) / 1e12,
        "value_graph_alternated": world * flops_step / (ms_graph_alt * 1e-3) / 1e12,
        other: world * flops_step / (ms_other * 1e-3) / 1e12,
        "speedup_vs_padded": base_ms["padded"] / base_ms["adaptive"],
        "speedup_vs_padded_no_unpad": base_ms["padded_no_unpad"] / base_ms["adaptive"],
        "padded_baseline": {"value": base_tf["padded"], "value_no_unpad": base_tf["padded_no_unpad"], "unit": UNIT,
                            "workspace_bytes": ws_bytes},
        "speedup_vs_padded_per_r": per_r,
        "memory_saved_pct": saved_pct,
        "memory_measured": mem_measured,
        "fp8_peak_frac": {"of_2x_measured_bf16": value / world / fp8_peak, "of_spec_4500": value / world / FP8_SPEC_TFLOPS},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": fp8_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp8_peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "peak_source": f"fp8 dense = 2 x bf16_tflops ({peaks_src})",
                     "kernel": f"tagg_gemm_kernel<2, 256, {int(args.exact)}, 1> (CTA pair, 256x256 tile)",
                     "traffic_source": "profiles/traffic_residual_sweep.json (ncu launch list, mean per launch)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "bound": "host link (PCIe)", "busier_direction_gbs": e2e_link_gbs,
                "note": "127 independent host-buffer calls per step: each copies its own A rows, A scales and group "
                        "sizes H2D (pinned) and its C rows D2H; expert weights resident; copies overlap the GEMMs "
                        "(hostpipe.run_host_batches)"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "extra": extra,
    }
    line["summary"] = summarize(line, fp8_peak)
    print(json.dumps(line), flush=True)
    print(line["summary"], file=sys.stderr, flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def summarize(line, fp8_peak):
    """<= 1 KB of the numbers that matter, for the stdout / stderr tails the driver keeps."""
    f = lambda x, d=0: "-" if x is None else f"{x:.{d}f}"  # noqa: E731
    out = [f"headline {f(line['value'])} TF/s ({f(100 * line['value'] / line['n_gpus'] / fp8_peak, 1)}% of "
           f"{fp8_peak:.0f}), eager {f(line.get('value_eager'))}, exact {f(line.get('value_exact'))}, "
           f"vs padded {f(line['speedup_vs_padded'], 2)}x (per-r min {f(line['speedup_vs_padded_per_r']['min'], 2)}x), "
           f"e2e {f(line['e2e']['value'])}, roofline {f(line['roofline']['frac'], 3)}"]
    cpu = line.get("cpu_baseline")
    if cpu:
        p = cpu.get("parity_vs_gpu_output") or {}
        out.append(f"cpu {f(cpu['value'], 3)} TF/s on {cpu['cores']} cores; self-check out_of_tol="
                   f"{p.get('out_of_tol')} bit_identical={f(p.get('bit_identical'), 4)}")
    ex = line.get("extra") or {}
    short = {"deepseek_v3_gateup_ep8_rank0": "DSv3 gu", "deepseek_v3_down_256e_1gpu": "DSv3 down",
             "qwen3_fwd_gateup": "Q3 fgu", "qwen3_fwd_down": "Q3 fdn", "qwen3_dgrad_down": "Q3 ddn",
             "qwen3_dgrad_gateup": "Q3 dgu"}
    cfgs = [f"{short[k]} {f(v['tflops'])} {f(100 * v['fp8_peak_frac'], 1)}% {f(v['speedup_vs_padded'], 2)}x "
            f"(burst {f(100 * v.get('fp8_peak_frac_burst'), 1) if v.get('fp8_peak_frac_burst') else '-'}%, sus "
            f"{f(100 * v.get('fp8_peak_frac_sustained'), 1) if v.get('fp8_peak_frac_sustained') else '-'}%)"
            for k, v in ex.items() if k in short and isinstance(v, dict) and "tflops" in v]
    if cfgs:
        out.append("; ".join(cfgs))
    sk = (ex.get("skinny_sweep") or {}).get("per_r")
    if sk:
        out.append("skinny " + " ".join(f"r{d['r']}:{f(d['us'], 1)}us/{f(100 * d['hbm_frac'])}%/"
                                        f"{f(d['speedup_vs_padded'], 2)}x" for d in sk))
    for k, lab in (("wgrad_dsv3_gateup", "wgrad"), ("moe_ffn_dsv3_1gpu", "moe fwd")):
        v = ex.get(k)
        if isinstance(v, dict) and "tflops" in v:
            out.append(f"{lab} {f(v['tflops'])} TF/s {f(100 * v['fp8_peak_frac'], 1)}%")
        if isinstance(v, dict) and isinstance(v.get("dy_block128"), dict):
            out.append(f"wgrad dY 128x128 {f(v['dy_block128']['tflops'])} TF/s "
                       f"{f(100 * v['dy_block128']['fp8_peak_frac'], 1)}%")
        if isinstance(v, dict) and isinstance(v.get("mxfp8"), dict):
            out.append(f"wgrad MXFP8 {f(v['mxfp8']['tflops'])} TF/s {f(100 * v['mxfp8']['fp8_peak_frac'], 1)}%")
    q = ex.get("quantize_dispatch_dsv3")
    if isinstance(q, dict) and "gbs" in q:
        out.append(f"quant+dispatch {f(q['gbs'])} GB/s {f(100 * q['hbm_frac'])}%")
    cq = ex.get("quantize_col_blocks_dsv3")
    if isinstance(cq, dict) and isinstance(cq.get("mxfp8"), dict):
        out.append(f"col quant {f(cq['fp32_scales']['gbs'])} GB/s {f(100 * cq['fp32_scales']['hbm_frac'])}% "
                   f"(MXFP8 {f(cq['mxfp8']['gbs'])} GB/s {f(100 * cq['mxfp8']['hbm_frac'])}%)")
    ep = ex.get("deepseek_v3_down_ep")
    if isinstance(ep, dict) and "gemm_tflops_aggregate" in ep:
        out.append(f"ep{ep['world']} gemm {f(ep['gemm_tflops_aggregate'])} TF/s e2e {f(ep['e2e_tflops_aggregate_incl_a2a'])}")
    return " | ".join(out)[:1024]


def burst_and_sustained(torch, fn, flops, trials=10, sustain_s=2.0):
    """The two timings MEASURED_PEAKS.json's bf16 roofs are taken with, applied to one launch
    of this kernel, so each fraction compares like with like: the BURST rate is the best of
    `trials` single launches (events around each, synchronized between them), against
    2 x bf16_tflops (best of 10); the SUSTAINED rate is launches back to back for `sustain_s`
    seconds (events around all), against 2 x bf16_tflops_sustained (4 s back to back).  The GEMM
    runs under sw_power_cap, so the clock -- and the rate -- fall as the run goes on."""
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(trials):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    n = max(3, int(sustain_s * 1e3 / best))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    sus = s.elapsed_time(e) / n
    return flops / (best * 1e-3) / 1e12, flops / (sus * 1e-3) / 1e12, n


def run_extra(torch, tg, dev, rank, fp8_peak, exact):
    """The other BASELINE.json configs on this GPU: TFLOP/s, speedup vs padded, memory saved.
    `tflops` is the mean of 5 back-to-back launches after 2 warm-ups (against the burst roof);
    `tflops_burst` / `tflops_sustained` follow the roofs' own timing (burst_and_sustained)."""
    peaks = _peaks()[0]
    fp8_sus = 2.0 * float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    out = {}
    specs = []
    _, local = deepseek_gateup_sizes(seed=0)
    specs.append(("deepseek_v3_gateup_ep8_rank0", [local], 4096, 7168, 32, "kn"))
    # DeepSeek-V3 down proj on one GPU: all 256 experts, 262,144 routed rows
    counts, _ = deepseek_gateup_sizes(seed=1)
    specs.append(("deepseek_v3_down_256e_1gpu", [counts], 7168, 2048, 256, "kn"))
    # Qwen3-235B-A22B: 128 experts, top-8 of 32768 tokens
    q, _ = deepseek_gateup_sizes(seed=2, experts=128, local=128)
    specs.append(("qwen3_fwd_gateup", [q], 3072, 4096, 128, "kn"))
    specs.append(("qwen3_fwd_down", [q], 4096, 1536, 128, "kn"))
    specs.append(("qwen3_dgrad_down", [q], 1536, 4096, 128, "nk"))
    specs.append(("qwen3_dgrad_gateup", [q], 4096, 3072, 128, "nk"))
    for name, sizes, n, k, G, layout in specs:
        P = Problem(torch, name, sizes, n, k, G, dev, seed=7 + rank, b_layout=layout)
        tf, ms, _ = run_problem_set(torch, tg, P, iters=5, warmup=2, exact=exact)
        gs = P.gs[0]
        burst, sus, n_sus = burst_and_sustained(
            torch, lambda: tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, b_layout=P.b_layout, out=P.out,
                                               exact_promotion=exact), sum(P.flops))
        acc = tg.account(P.sizes_list[0], n, k)
        out[name] = {"N": n, "K": k, "groups": G, "rows": sum(P.sizes_list[0]), "b_layout": layout,
                     "tflops": tf["adaptive"], "fp8_peak_frac": tf["adaptive"] / fp8_peak,
                     "padded_tflops": tf["padded"], "speedup_vs_padded": ms["padded"] / ms["adaptive"],
                     "speedup_vs_padded_no_unpad": ms["padded_no_unpad"] / ms["adaptive"],
                     "memory_saved_pct": acc.saving_pct, "ms": ms["adaptive"],
                     "tflops_burst": burst, "fp8_peak_frac_burst": burst / fp8_peak,
                     "tflops_sustained": sus, "fp8_peak_frac_sustained": sus / fp8_sus,
                     "sustained_launches": n_sus, "fp8_peak_sustained": fp8_sus}
        del P
        torch.cuda.empty_cache()
    out["quantize_dispatch_dsv3"] = run_quantize_dispatch(torch, tg, dev)
    out["quantize_col_blocks_dsv3"] = run_quantize_col_blocks(torch, tg, dev)
    out["wgrad_dsv3_gateup"] = run_wgrad(torch, tg, dev, fp8_peak)
    out["moe_ffn_dsv3_1gpu"] = run_moe_ffn(torch, tg, dev, fp8_peak)
    out["dense_fp8_reference_8192"] = run_dense_reference(torch, tg, dev, fp8_peak)
    out["skinny_sweep"] = run_skinny(torch, tg, dev)
    return out


def run_wgrad(torch, tg, dev, fp8_peak, iters=5, warmup=2):
    """dW_g = X_g^T dY_g for the DeepSeek-V3 gate+up shapes (32 local
    experts, skewed M_g, K=7168, N=4096): the ragged rows are the reduction axis.  Two dY
    recipes: per-(token block, column) scales (two packed ops per element pair in the
    promotion) and 128x128 block scales (one FFMA2 per pair, TAGG_WGRAD_DY_BLOCK128); and the
    MXFP8 recipe (per-(token block, column) power-of-two scales for X and dY, applied by the
    tensor core as E8M0 block scales with no promotion, TAGG_WGRAD_MX)."""
    _, sizes = deepseek_gateup_sizes(seed=0)
    sizes = [int(s) for s in sizes]
    m, k, n = sum(sizes), 7168, 4096
    gen = torch.Generator(device=dev).manual_seed(5)
    gs = torch.tensor(sizes, dtype=torch.int32, device=dev)
    x = torch.randn((m, k), device=dev, generator=gen).to(torch.bfloat16)
    dy = torch.randn((m, n), device=dev, generator=gen).to(torch.bfloat16)
    xc, xs = tg.quantize_col_blocks(x, gs)
    dw = torch.empty((len(sizes), k, n), dtype=torch.bfloat16, device=dev)
    flops = 2.0 * m * k * n
    res = {"groups": len(sizes), "rows": m, "K": k, "N": n, "dw_bytes": len(sizes) * k * n * 2,
           "tile": "CTA pair 256x256, cta_group::2"}
    xm, _, xf = tg.quantize_col_blocks_mx(x, gs)
    dm, _, dfac = tg.quantize_col_blocks_mx(dy, gs)
    for label, block, mx in (("per_column_dy", False, False), ("dy_block128", True, False), ("mxfp8", False, True)):
        if mx:
            fn = lambda: tg.wgrad_fp8_mx(xm, xf, dm, dfac, gs, out=dw)  # noqa: E731
        else:
            dc, ds = tg.quantize_col_blocks(dy, gs, block_cols=128 if block else 1)
            fn = lambda: tg.wgrad_fp8(xc, xs, dc, ds, gs, out=dw, dy_block128=block)  # noqa: E731
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        res[label] = {"ms": ms, "tflops": flops / ms / 1e9, "fp8_peak_frac": flops / ms / 1e9 / fp8_peak}
    # the headline keys: the per-column recipe (round 1's), then the block one beside it
    res.update({"ms": res["per_column_dy"]["ms"], "tflops": res["per_column_dy"]["tflops"],
                "fp8_peak_frac": res["per_column_dy"]["fp8_peak_frac"]})
    return res


def run_quantize_col_blocks(torch, tg, dev, rows=262144, cols=7168, groups=256, iters=5, warmup=2):
    """The weight gradient's column-block quantizer (HBM-bound) on the DeepSeek-V3 backward's
    grouped activations (262,144 routed rows of bf16 x 7168, 256 experts of 1024 rows): the
    per-column fp32-scale recipe and the MXFP8 recipe.  Algorithmic bytes = x read + codes
    written (the scales are 1/32 of the codes)."""
    peaks = _peaks()[0]
    gs = torch.full((groups,), rows // groups, dtype=torch.int32, device=dev)
    x = torch.randn((rows, cols), device=dev, generator=torch.Generator(device=dev).manual_seed(9)).to(torch.bfloat16)
    nbytes = rows * cols * 3
    res = {"rows": rows, "cols": cols, "groups": groups, "bytes": nbytes}
    for label, fn in (("fp32_scales", lambda: tg.quantize_col_blocks(x, gs)),
                      ("mxfp8", lambda: tg.quantize_col_blocks_mx(x, gs))):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        res[label] = {"ms": ms, "gbs": nbytes / ms / 1e6, "hbm_frac": nbytes / ms / 1e6 / float(peaks["hbm_gbs"])}
    del x
    torch.cuda.empty_cache()
    return res


def run_quantize_dispatch(torch, tg, dev, tokens=32768, k=7168, topk=8, experts=256, iters=10, warmup=3):
    """bf16 activations -> 1x128 FP8 codes + scales written straight
    into the expert-contiguous padding-free layout (route plan + fused quantize/scatter).
    HBM-bound: algorithmic bytes = x read + codes/scales/dest written + routing ids."""
    gen = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn((tokens, k), device=dev, generator=gen).to(torch.bfloat16)
    logits = torch.randn((tokens, experts), device=dev, generator=gen)
    eids = torch.topk(logits, topk, dim=1).indices.to(torch.int32)
    for _ in range(warmup):
        tg.quantize_dispatch(x, eids, experts)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        tg.quantize_dispatch(x, eids, experts)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    kb = -(-k // 128)
    rows = tokens * topk
    nbytes = tokens * k * 2 + rows * 4 + rows * (k + 4 * kb) + rows * 4 + experts * 4
    peak = _peaks()[0]["hbm_gbs"]
    return {"tokens": tokens, "K": k, "topk": topk, "experts": experts, "ms": ms,
            "algorithmic_bytes": nbytes, "gbs": nbytes / ms / 1e6, "hbm_frac": nbytes / ms / 1e6 / peak,
            "hbm_peak_gbs": peak, "note": "route plan (3 launches) + quantize/scatter (1 launch), x resident"}


def run_skinny(torch, tg, dev, iters=10):
    """SURVEY.md §8d, configs[1] variant "skinny": 8 groups of M_g = r rows (N=4096, K=7168,
    per-expert B [8, 7168, 4096]).  HBM-bound: every launch streams all of B (235 MB) for
    8r rows, so the roofline is achieved GB/s of the algorithmic bytes."""
    hbm = _peaks()[0]["hbm_gbs"]
    res = []
    for r in (1, 8, 32, 64, 127):
        P = Problem(torch, f"skinny_r{r}", [tuple([r] * 8)], 4096, 7168, 8, dev, seed=r)
        gs = P.gs[0]
        ws = tg.PaddedWorkspace(P.m_alloc, P.G, P.k, P.n, dev)

        def timed(fn):
            for _ in range(3):
                fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(iters):
                fn()
            e.record()
            torch.cuda.synchronize()
            return s.elapsed_time(e) / iters

        t = timed(lambda: tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out))
        tp = timed(lambda: tg.padded_grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, ws, out=P.out))
        nbytes = P.algorithmic_bytes(P.sizes_list[0])
        res.append({"r": r, "us": t * 1e3, "gbs": nbytes / t / 1e6, "hbm_frac": nbytes / t / 1e6 / hbm,
                    "tflops": P.flops[0] / (t * 1e-3) / 1e12, "speedup_vs_padded": tp / t})
        del P, ws
    return {"groups": 8, "N": 4096, "K": 7168, "hbm_peak_gbs": hbm, "per_r": res}


def run_dense_reference(torch, tg, dev, fp8_peak, n=8192, iters=10, warmup=3):
    """dense FP8 on the same box in the same run.  cuBLAS ``torch._scaled_mm``
    (e4m3, one scale per tensor, no per-block promotion) against this kernel on one 8192-row
    group with its 1x128 / 128x128 scales."""
    g = torch.Generator(device=dev).manual_seed(5)
    a = (torch.randn((n, n), device=dev, generator=g) * 0.5).to(torch.float8_e4m3fn)
    bt = (torch.randn((n, n), device=dev, generator=g) * 0.5).to(torch.float8_e4m3fn)
    one = torch.ones((), device=dev)
    sa = torch.rand((n, n // 128), device=dev, generator=g) * 1e-2 + 1e-3
    sb = torch.rand((1, n // 128, n // 128), device=dev, generator=g) * 1e-2 + 1e-3
    gs = torch.tensor([n], dtype=torch.int32, device=dev)
    b3 = bt.view(torch.uint8).view(1, n, n)
    out = torch.empty((n, n), dtype=torch.bfloat16, device=dev)

    def cublas():
        torch._scaled_mm(a, bt.t(), one, one, out_dtype=torch.bfloat16)

    def ours():
        tg.grouped_gemm_fp8(a, sa, b3, sb, gs, b_layout="nk", out=out)

    res = {}
    for name, fn in (("cublas_scaled_mm", cublas), ("this_kernel_blockwise", ours)):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        res[name + "_tflops"] = 2.0 * n ** 3 / (s.elapsed_time(e) / iters * 1e-3) / 1e12
    res["fp8_peak_used"] = fp8_peak
    res["note"] = "cuBLAS has per-tensor scales (no promotion); this kernel promotes per 128-K block"
    return res


def run_moe_ffn(torch, tg, dev, fp8_peak, tokens=32768, topk=8, experts=256, hidden=7168, inter=2048, iters=5,
                warmup=2):
    """The whole padding-free MoE FFN forward at DeepSeek-V3 scale on one GPU (all 256
    experts): quantize + dispatch -> GEMM gate|up -> SwiGLU + quantize -> GEMM down ->
    top-k combine.  Per-step device times from events on the one stream."""
    from paper_2508_16584_b200 import moe, quant

    g = torch.Generator(device=dev).manual_seed(11)
    x = torch.randn((tokens, hidden), device=dev, generator=g).to(torch.bfloat16)
    logits = torch.randn((tokens, experts), device=dev, generator=g)
    top = torch.topk(logits, topk, dim=1)
    eids = top.indices.to(torch.int32)
    wts = torch.softmax(top.values, dim=1)
    w = moe.ExpertWeights(_codes(torch, (experts, hidden, 2 * inter), g, dev),
                          _scales(torch, (experts, hidden // 128, 2 * inter // 128), g, dev),
                          _codes(torch, (experts, inter, hidden), g, dev),
                          _scales(torch, (experts, inter // 128, hidden // 128), g, dev))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    names = ("quantize_dispatch", "gemm_gate_up", "swiglu_quantize", "gemm_down", "combine")
    acc = [0.0] * 5

    def step(timed):
        if timed:
            ev[0].record()
        d = quant.quantize_dispatch(x, eids, experts)
        if timed:
            ev[1].record()
        h = tg.grouped_gemm_fp8(d.a_codes, d.a_scales, w.w_gate_up, w.s_gate_up, d.group_sizes)
        if timed:
            ev[2].record()
        a2, s2 = moe.swiglu_quantize(h, d.group_sizes)
        if timed:
            ev[3].record()
        c = tg.grouped_gemm_fp8(a2, s2, w.w_down, w.s_down, d.group_sizes)
        if timed:
            ev[4].record()
        y = moe.combine(c, d.dest_rows, wts)
        if timed:
            ev[5].record()
        return y

    for _ in range(warmup):
        step(False)
    torch.cuda.synchronize()
    for _ in range(iters):
        step(True)
        torch.cuda.synchronize()
        for i in range(5):
            acc[i] += ev[i].elapsed_time(ev[i + 1])
    ms = [a / iters for a in acc]
    rows = tokens * topk
    flops = 2.0 * rows * hidden * 2 * inter + 2.0 * rows * inter * hidden
    total = sum(ms)
    res = {"tokens": tokens, "topk": topk, "experts": experts, "hidden": hidden, "intermediate": inter,
           "ms": total, "tflops": flops / (total * 1e-3) / 1e12, "fp8_peak_frac": flops / (total * 1e-3) / 1e12 / fp8_peak,
           "breakdown_ms": dict(zip(names, ms)),
           "note": "all intermediates padding-free (no pad rows, no permutation between the GEMMs)"}
    # backward: dgrad of both GEMMs (K-major weights), SwiGLU backward (K9), wgrad (K6) of both,
    # dx via the combine, router-weight grads; 2x the forward FLOPs
    dy = torch.randn((tokens, hidden), device=dev, generator=g).to(torch.bfloat16)
    _, ctx = moe.moe_ffn(x, eids, wts, w, save=True)
    for _ in range(1):
        moe.moe_ffn_backward(dy, ctx, w)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bw_iters = 2
    s.record()
    for _ in range(bw_iters):
        grads = moe.moe_ffn_backward(dy, ctx, w)
    e.record()
    torch.cuda.synchronize()
    bw_ms = s.elapsed_time(e) / bw_iters
    marks = []
    grads = moe.moe_ffn_backward(dy, ctx, w, marks=marks)
    torch.cuda.synchronize()
    breakdown = {marks[i][0]: marks[i - 1][1].elapsed_time(marks[i][1]) for i in range(1, len(marks))}
    # the same backward with the other weight-gradient recipes (moe_ffn_backward(wgrad_recipe=))
    recipes = {}
    for recipe in ("dy_block128", "mxfp8"):
        moe.moe_ffn_backward(dy, ctx, w, wgrad_recipe=recipe)
        torch.cuda.synchronize()
        s.record()
        for _ in range(bw_iters):
            grads = moe.moe_ffn_backward(dy, ctx, w, wgrad_recipe=recipe)
        e.record()
        torch.cuda.synchronize()
        r_ms = s.elapsed_time(e) / bw_iters
        recipes[recipe] = {"ms": r_ms, "tflops": 2 * flops / (r_ms * 1e-3) / 1e12}
    del grads, ctx
    res["backward"] = {"ms": bw_ms, "tflops": 2 * flops / (bw_ms * 1e-3) / 1e12, "breakdown_ms": breakdown,
                       "wgrad_recipe": "per_column", "other_wgrad_recipes": recipes,
                       "dw_bytes": 2 * experts * hidden * 3 * inter,
                       "note": "dgrad x2 (b_layout nk), K9, wgrad x2 (K6, column-block quantized operands), "
                               "dx combine (K8), row gathers (K10), router grads (K11)"}
    return res


def run_ep_down(torch, dist, tg, dev, rank, world, fp8_peak, exact, iters=5, warmup=2):
    """BASELINE.json configs[3]: DeepSeek-V3 down proj (N=7168, K=2048), 256 experts
    sharded over the ranks, 32768 tokens x top-8 (strong scaling: each rank
    routes 32768/world tokens).  NCCL all_to_all dispatch of the FP8 rows +
    scales, then the padding-free grouped GEMM on the rank's experts.  Device
    time is measured with events and the max is taken over ranks."""
    from paper_2508_16584_b200 import ep

    E, N, K, topk, tokens = 256, 7168, 2048, 8, 32768
    epr = E // world
    t_local = tokens // world
    g = torch.Generator(device=dev).manual_seed(4242)  # same popularity map on every rank
    logp = -0.8 * torch.log(torch.randperm(E, device=dev, generator=g).float() + 1)
    gr = torch.Generator(device=dev).manual_seed(100 + rank)
    gumbel = -torch.log(-torch.log(torch.rand((t_local, E), device=dev, generator=gr).clamp_min(1e-20)))
    eid = torch.topk(logp[None, :] + gumbel, topk, dim=1).indices.reshape(-1)
    rows = eid.numel()
    a = _codes(torch, (rows, K), gr, dev)
    sa = _scales(torch, (rows, K // 128), gr, dev)
    b = _codes(torch, (epr, K, N), gr, dev)
    sb = _scales(torch, (epr, K // 128, N // 128), gr, dev)
    state = {}

    def dispatch():
        state["a"], state["sa"], state["meta"] = ep.dispatch(a, sa, eid, E, in_place=True)

    def gemm():
        m = state["a"].shape[0]
        if "out" not in state or state["out"].shape[0] < m:
            state["out"] = torch.empty((max(m, 1), N), dtype=torch.bfloat16, device=dev)
        if m:
            tg.grouped_gemm_fp8(state["a"], state["sa"], b, sb, state["meta"].group_sizes, out=state["out"],
                                exact_promotion=exact, b_index=state["meta"].b_index)

    def combine():
        m = state["a"].shape[0]
        state["back"] = ep.combine(state["out"][:m], state["meta"])

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # At world 1 there is no exchange to hide: one chunk on every SM (each further chunk would
    # re-read all of B).  Across GPUs, 4 chunks with 16 SMs left to the NCCL kernels.
    gemm_sms = sms if world == 1 else sms - 16
    chunks = 1 if world == 1 else 4

    def capped(codes, scales, gs, b_index=None, out=None):
        return tg.grouped_gemm_fp8(codes, scales, b, sb, gs, exact_promotion=exact, max_sms=gemm_sms,
                                   b_index=b_index, out=out)

    def overlapped():
        state["ov"] = ep.pipelined_expert_gemm(a, sa, eid, E, capped, N, chunks=chunks)

    for _ in range(warmup):
        dispatch()
        gemm()
        combine()
        overlapped()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    t_a2a = t_gemm = t_comb = t_ov = 0.0
    for _ in range(iters):
        ev[0].record()
        dispatch()
        ev[1].record()
        gemm()
        ev[2].record()
        combine()
        ev[3].record()
        torch.cuda.synchronize()
        dist.barrier()
        ev[4].record()
        overlapped()
        ev[5].record()
        torch.cuda.synchronize()
        t_a2a += ev[0].elapsed_time(ev[1])
        t_gemm += ev[1].elapsed_time(ev[2])
        t_comb += ev[2].elapsed_time(ev[3])
        t_ov += ev[4].elapsed_time(ev[5])
    same = bool(torch.equal(state["back"].view(torch.int16), state["ov"].view(torch.int16)))
    local_rows = state["a"].shape[0]
    flops_local = 2.0 * local_rows * N * K
    stats = torch.tensor([t_a2a / iters, t_gemm / iters, flops_local, local_rows, t_comb / iters, t_ov / iters],
                         dtype=torch.float64, device=dev)
    mx = stats.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    tot = stats.clone()
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    a2a_ms, gemm_ms, comb_ms, ov_ms = float(mx[0]), float(mx[1]), float(mx[4]), float(mx[5])
    seq_ms = a2a_ms + gemm_ms + comb_ms
    return {"N": N, "K": K, "experts": E, "experts_per_rank": epr, "tokens": tokens, "topk": topk, "world": world,
            "rows_total": int(tot[3]), "rows_max_rank": int(mx[3]),
            "gemm_tflops_aggregate": float(tot[2]) / (gemm_ms * 1e-3) / 1e12,
            "gemm_tflops_per_gpu_max_rank": float(mx[2]) / (gemm_ms * 1e-3) / 1e12,
            "e2e_tflops_aggregate_incl_a2a": float(tot[2]) / ((gemm_ms + a2a_ms) * 1e-3) / 1e12,
            "a2a_ms_max": a2a_ms, "gemm_ms_max": gemm_ms, "combine_ms_max": comb_ms,
            "sequential_dispatch_gemm_combine_ms": seq_ms,
            "overlapped": {"ms": ov_ms, "chunks": chunks, "gemm_sms": gemm_sms,
                           "tflops_aggregate": float(tot[2]) / (ov_ms * 1e-3) / 1e12,
                           "speedup_vs_sequential": seq_ms / ov_ms, "bitwise_equal_to_sequential": same},
            "a2a_bytes_per_row": K + 4 * (K // 128), "transport": "NCCL all_to_all_single (NVLink/NVSwitch)"}


if __name__ == "__main__":
    main()

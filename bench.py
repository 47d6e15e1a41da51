"""Benchmark of the Sample-Align-D hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl mine|reference]

A step is one pass of the whole hot path over one batch of synthetic input
(DESIGN.md §7): S1 profiles, S2a local ranks, S2b samples, S2c sample
exchange, S2d global ranks, S3 pivots and buckets, S4 redistribution, S1' the
received profiles, S5 every bucket's all-pairs similarity matrix.  Under
torchrun each rank (one per GPU) holds p/N logical blocks and owns p/N buckets;
collectives go through torch.distributed (NCCL).  Rank 0 prints one JSON line.

value   = k-mer similarity sequence-pairs evaluated per second by the whole job
          (S2a + S2d + S5 pairs, SURVEY §8(d) accounting) / max-over-ranks time
          of K device-timed steps, inputs resident in HBM;
e2e     = the same through the public API with the step's inputs copied from
          pinned host memory and its results (buckets, member ids, every
          bucket's uint16 numerator and fp64 similarity matrices as packed
          upper triangles) copied back inside the timed region (consecutive
          steps pipelined: step t+1 computes while step t's results copy);
          e2e.numerators_only = the same without the fp64 matrices;
roofline= the dominant kernel (the S5 GEMM): the method's work (2 x 8000 ops
          per pair, Eq. 1) against the e2m1 tensor peak, and its algorithmic
          HBM bytes (full C + F output, operand rows once) against the copy
          bandwidth; `bound` is the binding one;
cpu_baseline = the CPU oracle (oracle/, as it stands) on a bounded sample of
          the same workload, on the host's cores (rank 0, N = 1 only).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "k-mer similarity sequence-pairs/s and partition time at 1/2/4/8 B200; % roofline"
UNIT = "sequence-pairs/s"
EPS_BINS = 8000                      # 20^3 bin-ops per pair (Eq. 1)
# ALU-pipe bound of the dense min-sum: 2 warp-instr/clk/SM x 32 lanes x bins per instruction
BINOPS_PER_SM_CLK = {"u8": 256,       # VABSDIFF4.U8.ACC: 4 bins (sum|a-b| identity)
                     "u16": 128,      # VIMNMX.U16x2: 2 bins (adds also on the ALU pipe: 85 reachable)
                     "u16imad": 128}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def workload_desc(cfg):
    L = cfg.length
    ln = (f"ancestor length U[{L[1]},{L[2]}]" if L[0] == "uniform"
          else f"lengths lognormal mean {L[1]} sigma {L[2]} clipped [{L[3]},{L[4]}]")
    return (f"{cfg.name}: N={cfg.n} protein seqs, {cfg.families} families, {ln}, "
            f"{int(cfg.p_sub * 100)}% subst + {int(cfg.p_indel * 100)}% indel, k={cfg.k}, p={cfg.p}, "
            f"{cfg.samples_per_block} samples per block")


# ------------------------------------------------------------ clocks -----
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 100):
        self.index = index
        self.period_ms = period_ms
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 10.0):
        """Block until nvidia-smi delivers its first sample: its start-up (NVML
        initialisation, driver locks) must not overlap the timed region."""
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)
        time.sleep(0.15)   # past the first sample's query as well

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, pw = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
                pw.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# -------------------------------------------------------- CPU oracle ------
def cpu_oracle_sample(ds, cfg, n_sample: int, workers: int):
    """The oracle (as it stands) on the first n_sample sequences of the
    workload, partitioned with the workload's p and k_b (capped at the block
    size) plus every bucket's similarity matrix.  Returns (pairs, seconds)."""
    from oracle import kmer, partition
    sub = ds.subset(np.arange(n_sample))
    t0 = time.perf_counter()
    P, nk = kmer.profiles(sub.residues, sub.offsets, cfg.k, cfg.alphabet)
    w = n_sample // cfg.p
    kb = min(cfg.samples_per_block, w)
    r = partition.partition(P, nk, cfg.p, kb, workers=workers)
    s5 = 0
    for mem in r.buckets:
        if len(mem):
            partition.bucket_similarity(P, nk, mem, workers=workers)
            s5 += len(mem) * (len(mem) - 1) // 2
    dt = time.perf_counter() - t0
    bounds = partition.block_bounds(n_sample, cfg.p)
    s2a = sum((bounds[q + 1] - bounds[q]) * (bounds[q + 1] - bounds[q] - 1) // 2 for q in range(cfg.p))
    s2d = n_sample * cfg.p * kb
    return s2a + s2d + s5, dt, kb


def run_reference(args, cfg, ds):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import kmer
    workers = kmer.default_workers()
    n_s = args.cpu_sample_n
    for _ in range(args.warmup):
        cpu_oracle_sample(ds, cfg, n_s, workers)
    tot_pairs, tot_s = 0, 0.0
    for _ in range(args.steps):
        pairs, dt, kb = cpu_oracle_sample(ds, cfg, n_s, workers)
        tot_pairs += pairs
        tot_s += dt
    v = tot_pairs / tot_s
    sample = (f"oracle profiles + Alg.2 partition (p={cfg.p}, k_b={kb}) + all bucket matrices on the first "
              f"{n_s} sequences of {cfg.name}, per step")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64/f64 (numpy)",
            "data": "synthetic", "config": {"workload": workload_desc(cfg), "reference_sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm ----
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--prewarm-s", type=float, default=0.3,
                    help="seconds of untimed dense matmuls before the warm-up steps (GPU power state)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=2400)
    ap.add_argument("--no-similarity", action="store_true", help="S5 numerators only (not the default)")
    ap.add_argument("--clock-period-ms", type=int, default=100,
                    help="nvidia-smi sampling period during the timed region")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "torch"],
                    help="N > 1: libsa's NCCL communicator (default) or torch.distributed callbacks")
    args = ap.parse_args()

    from sa_synth.generator import CONFIGS, generate
    cfg = CONFIGS[args.config]
    ds = generate(cfg)
    if args.impl == "reference":
        run_reference(args, cfg, ds)
        return

    import torch
    import torch.distributed as dist

    from paper_0905_1744_b200 import binding as B
    from paper_0905_1744_b200.pipeline import HotPath, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if cfg.p % world:
        raise SystemExit(f"p={cfg.p} is not divisible by {world} GPUs")

    first, last = shard_range(ds.n, cfg.p, world, rank)
    r0, r1 = int(ds.offsets[first]), int(ds.offsets[last])
    res_h = torch.from_numpy(ds.residues[r0:r1].copy()).pin_memory()
    offs_h = torch.from_numpy(ds.offsets[first:last + 1] - ds.offsets[first]).pin_memory()
    res_d = res_h.to(dev)
    offs_d = offs_h.to(dev)

    ctx = B.Context(local)
    if world > 1:
        if args.comm == "nccl":   # libsa's own NCCL communicator: no Python in any collective
            obj = [B.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx.attach_nccl(obj[0], world, rank)
        else:                     # torch.distributed callbacks (sa_comm_ops)
            ctx.attach_comm(B.TorchComm(device=dev))
    ctx.set_timing(True)
    hp = HotPath(ctx, cfg.p, cfg.samples_per_block, want_similarity=not args.no_similarity)
    # every step runs on a dedicated (non-default) stream, so the e2e leg's
    # copy stream is not serialised against it by legacy-stream semantics
    st = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(st)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    names = ["start", "S1", "S4", "S1b", "S5"]
    # bring the GPU out of its idle power state before the warm-up steps (a
    # fresh box's first steps ran at half speed otherwise): ~0.3 s of dense
    # matmuls on the step stream, untimed, no part of the workload
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    t_end = time.perf_counter() + args.prewarm_s
    while time.perf_counter() < t_end:
        for _ in range(20):
            a = torch.tanh(a @ a)
        torch.cuda.synchronize()
    del a
    for _ in range(args.warmup):
        out = hp.step(res_d, offs_d, ds.n, first)
    torch.cuda.synchronize()
    ctx.set_timing(True)   # clears the phase history: it now holds the timed steps only

    # ------------------------------------------------ device-timed steps
    per_step = []
    clocks = ClockSampler(local, period_ms=args.clock_period_ms)
    # no garbage-collector pause inside a timed region (the step has one host
    # block, C3, and its post-C3 launches keep the GPU fed only while the host
    # thread runs: a collection there is a GPU-idle gap)
    gc.collect()
    gc.disable()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    clocks.wait_first()
    for _ in range(int(os.environ.get("SA_BENCH_SETTLE_STEPS", "0"))):   # diagnostics: untimed steps after the sampler's start-up
        hp.step(res_d, offs_d, ds.n, first)
    torch.cuda.synchronize()
    launches0 = B.sa_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # every step's events exist before the timed region (torch creates the CUDA
    # event at its first record): no event creation inside the timed loop
    pre = [{k: torch.cuda.Event(enable_timing=True) for k in names} for _ in range(args.steps)]
    if os.environ.get("SA_BENCH_LAZY_EVENTS", "0") != "1":
        for d in pre:
            for e in d.values():
                e.record(st)
        torch.cuda.synchronize()
    e0.record(st)
    for i in range(args.steps):
        # no host synchronisation inside the timed region: libsa only records
        # its phase events; they are read after the region (phase_history)
        ev = pre[i]
        ev["_host"] = []
        out = hp.step(res_d, offs_d, ds.n, first, events=ev)
        per_step.append(ev)
    e1.record(st)
    torch.cuda.synchronize()
    launches = B.sa_launch_count() - launches0
    gc.enable()
    barrier()
    clk = clocks.stop()
    total_ms = max_over_ranks(e0.elapsed_time(e1))
    hist = {k: ctx.phase_history(k)[-args.steps:] for k in B.PHASES}
    per_step = [(ev, {k: (hist[k][i] if i < len(hist[k]) else 0.0) for k in B.PHASES})
                for i, ev in enumerate(per_step[-len(hist["S2a"]):] if hist["S2a"] else per_step)]

    # pair accounting; bucket sizes are known on every rank
    bounds = [q * ds.n // cfg.p for q in range(cfg.p + 1)]
    s2a_pairs = sum((bounds[q + 1] - bounds[q]) * (bounds[q + 1] - bounds[q] - 1) // 2 for q in range(cfg.p))
    s2d_pairs = ds.n * cfg.p * cfg.samples_per_block
    sizes = out.part.counts.sum(axis=0)
    s5_pairs = int(sum(int(n) * (int(n) - 1) // 2 for n in sizes))
    pairs = s2a_pairs + s2d_pairs + s5_pairs
    value = pairs * args.steps / (total_ms / 1e3)

    def med(f):
        return statistics.median(f(ev, ph) for ev, ph in per_step)

    part_ms = med(lambda ev, ph: ev["S1"].elapsed_time(ev["S4"]))
    s5_ms = med(lambda ev, ph: ev["S1b"].elapsed_time(ev["S5"]))
    phases = {
        "S1": med(lambda ev, ph: ev["start"].elapsed_time(ev["S1"])),
        "S2a": med(lambda ev, ph: ph["S2a"]), "S2b": med(lambda ev, ph: ph["S2b"]),
        "S2c": med(lambda ev, ph: ph["S2c"]), "S2d": med(lambda ev, ph: ph["S2d"]),
        "S3": med(lambda ev, ph: ph["S3"]),
        "partition_S2a_to_S4": part_ms,
        "S1_received": med(lambda ev, ph: ev["S4"].elapsed_time(ev["S1b"])),
        "S5": s5_ms,
        "S5_gemm": med(lambda ev, ph: ph["gemm_S5"]),
        "S2a_gemm": med(lambda ev, ph: ph["gemm_S2a"]),
        "S2d_gemm": med(lambda ev, ph: ph["gemm_S2d"]),
    }
    part_ms_max = max_over_ranks(part_ms)
    s5_ms_max = max_over_ranks(s5_ms)

    # roofline of the dominant kernel: K2 over this rank's S5 launches
    peaks, peak_src = load_peaks()
    sm_mhz_peak = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    engine = ctx.engine()
    own = list(B.owned_buckets(cfg.p, world, rank))
    my_s5_pairs = sum(int(sizes[b]) * (int(sizes[b]) - 1) // 2 for b in own)
    traffic = None
    if engine == "tc":
        # K2T: the S5 buckets as exact 0/1 contractions on the
        # tensor cores.  The roofline counts the METHOD's work, not the
        # implementation's contraction: Eq. 1 is EPS_BINS = 8000 min-accumulate
        # bin-ops per pair, each one e2m1 multiply-add (2 ops) -- so
        # 2 * 8000 * pairs ops -- against the e2m1 tensor peak; the kernel must
        # also write the full symmetric C (uint16) and F (fp64) of every bucket
        # and read each bucket's operand rows once: that HBM floor is the other
        # roofline.  `bound` is whichever floor is larger (the binding one);
        # both fractions are reported, and the implementation's own contraction
        # length K' (kept threshold-layer columns) as a secondary figure.
        nz = [(b, row, n_b) for b, row, n_b in out.buckets if n_b > 0]
        rb_s5 = [r for _, r, _ in out.buckets] + [sum(n for _, _, n in out.buckets)]
        B.sa_bucket_similarity_batch(ctx, out.bucket_profiles, out.bucket_nkmers, rb_s5, hp.bins,
                                     numerators=out.numerators, similarity=out.similarity)
        kcols = dict(zip([b for b, _, _ in nz], ctx.tc_columns()))
        operand = ctx.tc_operand()
        gemm_ms = phases["S5_gemm"]
        bf16 = float(peaks.get("bf16_tflops", 1590.0))
        ratio = 4.0 if operand == "e2m1" else 2.0   # nominal dense 9 (fp4) / 4.5 (int8) vs 2.25 (bf16) PF
        peak_t = ratio * bf16 * 1e12
        ops_method = 2.0 * EPS_BINS * my_s5_pairs
        ops_kprime = sum(2.0 * kcols[b] * int(sizes[b]) * (int(sizes[b]) - 1) / 2 for b in kcols)
        hbm = float(peaks.get("hbm_gbs", 6551.0)) * 1e9
        out_bytes = sum(int(sizes[b]) ** 2 * ((2 if hp.want_num else 0) + (8 if hp.want_sim else 0)) for b in own)
        opnd_bytes = sum(int(sizes[b]) * (EPS_BINS // 2 if operand == "e2m1" else EPS_BINS) for b in own)
        bytes_alg = out_bytes + opnd_bytes
        t_tensor = ops_method / peak_t
        t_hbm = bytes_alg / hbm
        tpath = os.path.join(ROOT, "profiles", "k2t_traffic.json")
        ncu_note = None
        if os.path.exists(tpath):
            with open(tpath) as f:
                tj = json.load(f)
            if tj.get("operand", "u8") == operand:
                traffic = tj.get("dram_bytes_per_launch")
                ncu_note = {k: tj[k] for k in ("tensor_active_pct", "source", "round") if k in tj}
        cta_pairs = os.environ.get("SA_K2T_PAIR", "1") != "0"
        kernel = (f"tc::{'gemm2_kernel' if cta_pairs else 'gemm_kernel'}<KeyMatEpi<NUM|SIM>> (K2T, "
                  f"{'tcgen05 cta_group::2 CTA pairs' if cta_pairs else 'one CTA per tile'}, {operand} operands, "
                  f"S5 bucket matrices, one launch per step)")
        common = {"kernel": kernel, "engine": engine, "operand": operand, "kernel_ms": gemm_ms, "traffic": traffic,
                  "frac_tensor_method": t_tensor * 1e3 / gemm_ms, "frac_hbm": t_hbm * 1e3 / gemm_ms,
                  "frac_tensor_kprime": ops_kprime / peak_t * 1e3 / gemm_ms,
                  "kprime": [kcols[b] for b in sorted(kcols)],
                  "tensor_peak_source": (f"{peak_src} bf16_tflops {bf16:.1f} (burst, MEASURED_PEAKS.json) x "
                                         f"{ratio:.0f} = {'e2m1 (kind::mxf4)' if operand == 'e2m1' else 'u8 (kind::i8)'}"
                                         f" dense (nominal {'9' if operand == 'e2m1' else '4.5'} / 2.25 PF ratio)"),
                  "hbm_peak_source": f"{peak_src} hbm_gbs {hbm / 1e9:.1f} (MEASURED_PEAKS.json copy bandwidth)",
                  "algorithmic": (f"tensor: 2 x {EPS_BINS} ops per pair (Eq. 1 bins) x {my_s5_pairs} pairs; "
                                  f"hbm: full symmetric C (2 B) + F (8 B) per ordered pair "
                                  f"({out_bytes / 1e9:.3f} GB) + each bucket's e2m1 layer-1 operand rows once "
                                  f"({opnd_bytes / 1e9:.3f} GB); over the GEMM kernel's CUDA-event time "
                                  f"(median of the timed steps)"),
                  "phase_frac_tensor_method": t_tensor * 1e3 / s5_ms, "ncu": ncu_note}
        # the S5 floor is nearly all writes: against the write-only fill rate
        # measured on this GPU type (tools/hbm_write_probe.py) as well
        wpath = os.path.join(ROOT, "profiles", "r02s3_hbm_probe.jsonl")
        if os.path.exists(wpath):
            with open(wpath) as f:
                wfill = max(json.loads(l)["write_only_gbs"] for l in f if l.strip()) * 1e9
            common["frac_hbm_vs_write_fill"] = bytes_alg / wfill * 1e3 / gemm_ms
            common["write_fill_gbs"] = wfill / 1e9
        if t_hbm >= t_tensor:
            roof = {"bound": "hbm", "achieved": bytes_alg / (gemm_ms / 1e3) / 1e9, "peak": hbm / 1e9,
                    "unit": "GB/s", "frac": t_hbm * 1e3 / gemm_ms, **common}
        else:
            roof = {"bound": "tensor", "achieved": ops_method / (gemm_ms / 1e3) / 1e12, "peak": peak_t / 1e12,
                    "unit": "TOP/s", "frac": t_tensor * 1e3 / gemm_ms, **common}
    else:
        per_clk = BINOPS_PER_SM_CLK[engine]
        peak_binops = per_clk * nsm * sm_mhz_peak * 1e6
        achieved = my_s5_pairs * EPS_BINS / (s5_ms / 1e3)
        tpath = os.path.join(ROOT, "profiles", "k2_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        roof = {"bound": "alu", "kernel": f"minsum_kernel<sym, {engine}> (K2, S5 bucket matrices)",
                "engine": engine,
                "achieved": achieved / 1e12, "peak": peak_binops / 1e12, "unit": "Tbin-op/s",
                "frac": achieved / peak_binops, "traffic": traffic,
                "peak_source": (f"derived ({peak_src} sm_max_mhz): {per_clk} bin-ops/clk/SM = ALU pipe 2 warp-"
                                f"instr/clk/SM (ncu sm__inst_executed_pipe_alu peak) x 32 lanes x {per_clk // 64} "
                                f"bins per {'VABSDIFF4.U8.ACC' if engine == 'u8' else 'VIMNMX.U16x2'} x {nsm} SMs "
                                f"x {sm_mhz_peak:.0f} MHz"),
                "algorithmic": f"{EPS_BINS} bin-ops per pair x {my_s5_pairs} pairs / S5 CUDA-event time"}

    # ------------------------------------- partition: GEMM rooflines, collectives
    # The partition's dominant kernels are the two key GEMMs (S2a: every pair
    # of each local block, S2d: every local sequence against the s samples);
    # their method count is Eq. 1's 8000 bins per pair, as for S5.  Their
    # outputs are 128-bit keys (no HBM floor to speak of): the tensor floor binds.
    partition_roofline = None
    if engine == "tc":
        my_blocks = range(rank * cfg.p // world, (rank + 1) * cfg.p // world)
        my_s2a = sum((bounds[q + 1] - bounds[q]) * (bounds[q + 1] - bounds[q] - 1) // 2 for q in my_blocks)
        my_s2d = (bounds[my_blocks.stop] - bounds[my_blocks.start]) * cfg.p * cfg.samples_per_block
        partition_roofline = {"bound": "tensor", "unit": "TOP/s", "peak": peak_t / 1e12,
                              "peak_source": "as roofline.tensor_peak_source"}
        for name, pr, ms in (("S2a_gemm", my_s2a, phases["S2a_gemm"]), ("S2d_gemm", my_s2d, phases["S2d_gemm"])):
            ops = 2.0 * EPS_BINS * pr
            partition_roofline[name] = {"pairs": int(pr), "kernel_ms": ms, "achieved": ops / (ms / 1e3) / 1e12,
                                        "frac": ops / peak_t * 1e3 / ms}
        ops_all = 2.0 * EPS_BINS * (my_s2a + my_s2d)
        partition_roofline["partition_ms"] = part_ms
        partition_roofline["frac_of_partition_time"] = ops_all / peak_t * 1e3 / part_ms
    # Bytes each rank sends per step in the paper's exchanges (Alg. 2, P:1248-1267;
    # DESIGN.md §6), from this step's sizes: C1 sample broadcast (profiles + nk +
    # ids of the rank's s/G samples, allgather), C2 regular samples (32-byte
    # records), C3 count exchange (2p + 3 int64 per rank), C4 all-to-all: the
    # residues and 16-byte records of the rank's sequences whose bucket another
    # rank owns.  At N = 1 nothing leaves the GPU.
    stride = B.sa_profile_stride(hp.bins)
    s_loc = cfg.p // world * cfg.samples_per_block
    nb = np.asarray(out.part.bytes)
    nc = np.asarray(out.part.counts)
    own_of = [b * world // cfg.p for b in range(cfg.p)]
    c4_seq = int(sum(nc[rank, b] for b in range(cfg.p) if own_of[b] != rank))
    c4_bytes = int(sum(nb[rank, b] for b in range(cfg.p) if own_of[b] != rank)) + 16 * c4_seq
    sent = {"C1_sample_allgather": s_loc * (stride * 2 + 4 + 8),
            "C2_regular_samples_allgather": (cfg.p // world) * (cfg.p - 1) * 32,
            "C3_count_allgather": (2 * cfg.p + 3) * 8,
            "C4_alltoallv": c4_bytes}
    collectives = {"n_ranks": world, "bytes_sent_per_rank_per_step": sent if world > 1 else {k: 0 for k in sent},
                   "bytes_if_sharded_over_8": None}
    if world == 1 and cfg.p % 8 == 0:
        # what rank 0 would send at G = 8 (same data): C1 and C2 scale with the
        # rank's blocks; C4 is 7/8 of its sequences' residues + records
        g = 8
        blk = [q * ds.n // cfg.p for q in range(cfg.p + 1)]
        res_b = np.diff(ds.offsets)
        r0 = range(0, cfg.p // g)
        mine = np.arange(blk[r0.start], blk[r0.stop])
        bo = out.part.bucket_of.cpu().numpy()[mine]
        off = np.array([b * g // cfg.p != 0 for b in bo], dtype=bool)
        collectives["bytes_if_sharded_over_8"] = {
            "C1_sample_allgather": (cfg.p // g) * cfg.samples_per_block * (stride * 2 + 4 + 8),
            "C2_regular_samples_allgather": (cfg.p // g) * (cfg.p - 1) * 32,
            "C3_count_allgather": (2 * cfg.p + 3) * 8,
            "C4_alltoallv": int(res_b[mine][off].sum() + 16 * off.sum())}

    # --------------------------------------------- end-to-end (host buffers)
    def run_e2e(with_sim: bool):
        """K steps through the public API with host buffers: each step's
        residues are copied from pinned host memory, and its results -- bucket
        ids, received member ids, every owned bucket's numerator matrix and
        (with_sim) its fp64 similarity matrix, each as its packed upper
        triangle (the whole symmetric content) -- are copied back to pinned
        host memory inside the timed region."""
        h_out = {}
        # two copy streams, alternating by bucket: two copy engines share the PCIe link
        copy_sts = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]

        def pinned(k, t):
            if k not in h_out or h_out[k].shape != t.shape or h_out[k].dtype != t.dtype:
                h_out[k] = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            return h_out[k]

        # packed triangles double-buffered by step parity: step t + 1's S1-S4
        # (and its buckets' S5) overlap step t's copies; a buffer is reused
        # only after the copy that read it two steps earlier has finished
        d_packed, copied = {}, {}
        parity = [0]

        def ship(kind, b, mat, pack_fn, dtype):
            n_b = mat.shape[0]
            key = (parity[0], kind, b)
            if key not in d_packed or d_packed[key].numel() != n_b * (n_b + 1) // 2:
                d_packed[key] = torch.empty(n_b * (n_b + 1) // 2, dtype=dtype, device=dev)
            if key in copied:
                st.wait_event(copied[key])
            pk = pack_fn(ctx, mat, d_packed[key], stream=st)
            ev = torch.cuda.Event()
            ev.record(st)
            copy_st = copy_sts[b % 2]
            copy_st.wait_event(ev)
            with torch.cuda.stream(copy_st):
                src = pk.view(torch.int16) if dtype == torch.uint16 else pk
                pinned(f"{kind}{b}", src).copy_(src, non_blocking=True)
                copied[key] = torch.cuda.Event()
                copied[key].record(copy_st)

        def on_bucket(b, num, sim):
            # bucket b's matrices go to the host on a copy stream while the next bucket computes
            if num is not None:
                ship("num", b, num, B.sa_pack_upper_u16, torch.uint16)
            if with_sim and sim is not None:
                ship("sim", b, sim, B.sa_pack_upper_f64, torch.float64)

        def d2h_tail(o, last: bool):
            # on a copy stream too: a device-to-host copy on the step's stream
            # would hold the next step's kernels behind the copy engine's queue
            nb = 0
            ev = torch.cuda.Event()
            ev.record(st)
            copy_sts[0].wait_event(ev)
            with torch.cuda.stream(copy_sts[0]):
                for k, t in (("bucket_of", o.part.bucket_of), ("gid", o.recv_global_idx)):
                    t.record_stream(copy_sts[0])   # not reused by the allocator before the copy ran
                    pinned(k, t).copy_(t, non_blocking=True)
                    nb += t.numel() * t.element_size()
            for num, sim in zip(o.numerators, o.similarity):
                if num is not None:
                    nb += num.shape[0] * (num.shape[0] + 1) // 2 * 2
                if with_sim and sim is not None:
                    nb += sim.shape[0] * (sim.shape[0] + 1) // 2 * 8
            parity[0] ^= 1
            if last:
                for cs in copy_sts:
                    st.wait_stream(cs)       # the run ends when every step's results are on the host
            return nb

        res_dd = torch.empty_like(res_d)
        offs_dd = torch.empty_like(offs_d)
        for _ in range(2):   # allocate both parities' buffers and the pinned host buffers untimed
            o = hp.step(res_d, offs_d, ds.n, first, on_bucket=on_bucket)
            d2h_tail(o, last=True)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()
        f0.record(st)
        d2h_bytes = 0
        for i in range(args.steps):
            res_dd.copy_(res_h, non_blocking=True)
            offs_dd.copy_(offs_h, non_blocking=True)
            o = hp.step(res_dd, offs_dd, ds.n, first, on_bucket=on_bucket)
            d2h_bytes = d2h_tail(o, last=i == args.steps - 1)
        f1.record(st)
        torch.cuda.synchronize()
        gc.enable()
        e2e_ms = max_over_ranks(f0.elapsed_time(f1))
        del d_packed, h_out
        what = ("bucket_of, received member ids, and every owned bucket's symmetric uint16 numerator matrix "
                + ("and fp64 similarity matrix, each " if with_sim else "") +
                "as its packed upper triangle (sa_pack_upper_u16" + (" / _f64)" if with_sim else ")"))
        return {"value": pairs * args.steps / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(res_h.numel() + offs_h.numel() * 8),
                "d2h_bytes_per_step": int(d2h_bytes), "ms_per_step": e2e_ms / args.steps,
                "results_copied": what,
                "overlap": "steps pipelined: step t+1 computes while step t's triangles copy (double-buffered)"}

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(with_sim=hp.want_sim)
        if hp.want_sim:
            e2e["numerators_only"] = run_e2e(with_sim=False)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import kmer
        workers = kmer.default_workers()
        cp, cs, kb = cpu_oracle_sample(ds, cfg, args.cpu_sample_n, workers)
        cpu = {"value": cp / cs, "unit": UNIT, "cores": workers, "kind": "oracle",
               "sample": (f"oracle profiles + Alg.2 partition (p={cfg.p}, k_b={kb}) + all bucket matrices on "
                          f"the first {args.cpu_sample_n} sequences of {cfg.name}: {cp} pairs in {cs:.1f} s")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": (("e2m1 (0/1 threshold layers, f32 accumulate, exact)" if ctx.tc_operand() == "e2m1"
                       else "u8 (0/1 threshold layers, s32 accumulate)") if engine == "tc"
                      else {"u8": "u8"}.get(engine, "u16")),
            "data": "synthetic (seeded star-phylogeny protein families, sa_synth)",
            "config": {"workload": workload_desc(cfg), "N": ds.n, "p": cfg.p,
                       "samples_per_block": cfg.samples_per_block, "k": cfg.k, "alphabet": cfg.alphabet,
                       "dataset_sha256": ds.sha256(), "parallelism": f"{world} rank(s), {cfg.p // world} "
                       "blocks/buckets each",
                       "l2": "inputs larger than L2 (profiles N x 16 KB = "
                             f"{ds.n * 16000 / 1e9:.2f} GB per step)",
                       "prewarm_s": args.prewarm_s},
            "partition_ms": part_ms_max, "s5_ms": s5_ms_max,
            "pairs_per_step": {"S2a": s2a_pairs, "S2d": s2d_pairs, "S5": s5_pairs},
            "s5_pairs_per_s": s5_pairs / (s5_ms_max / 1e3),
            # rank-0 views of the other rows of the BASELINE.md reporting template
            "s2_pairs_per_s_rank0": (s2a_pairs + s2d_pairs) / world / ((phases["S2a"] + phases["S2d"]) / 1e3),
            "s1_hbm_rank0": {
                "bytes": int(res_h.numel() + offs_h.numel() * 8 + (last - first) * (16000 + 4)),
                "ms": phases["S1"],
                "frac_of_hbm": (res_h.numel() + offs_h.numel() * 8 + (last - first) * 16004) /
                               (phases["S1"] / 1e3) / (float(peaks.get("hbm_gbs", 6551.0)) * 1e9)},
            "phases_ms_rank0": phases,
            # device time between one step's last event and the next step's
            # first (per step, rank 0): the GPU waiting for the host to enqueue
            "inter_step_gap_ms_rank0": max(0.0, total_ms / args.steps - (phases["S1"] + part_ms + phases["S1_received"]
                                                                       + s5_ms)),
            # each timed step's device time, first event to last (rank 0): an
            # outlier step shows here (a host stall between C3 and S4)
            "step_ms_rank0": [round(ev["start"].elapsed_time(ev["S5"]), 3) for ev, _ in per_step],
            # host time of each step's enqueue segments (start -> S1 -> S4 -> S1b -> S5 marks), ms:
            # a device-side outlier with a long host segment is a host stall
            "host_segments_ms_rank0": [[round((b[1] - a[1]) * 1e3, 3) for a, b in zip(ev["_host"], ev["_host"][1:])]
                                       for ev, _ in per_step],
            # device time of the step's segments between the same marks, and of libsa's phases, per step
            "device_segments_ms_rank0": [[round(ev[a].elapsed_time(ev[b]), 3) for a, b in zip(names, names[1:])]
                                         for ev, _ in per_step],
            "phase_steps_ms_rank0": {k: [round(ph[k], 3) for _, ph in per_step] for k in ("S2a", "S2b", "S2c", "S2d", "S3")},
            "bucket_sizes": [int(x) for x in sizes],
            "exact_fallbacks": out.part.exact_fallbacks,
            "roofline": roof, "partition_roofline": partition_roofline, "collectives": collectives,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: synchronous Downpour training samples/s on B200 (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one synchronous Downpour round of the SPEC benchmark net
`lstm(5,20,10),softmax(20,3)`: every worker gathers its batch of
B=1000 samples from its HBM-resident shard, runs forward+loss+backward, the
gradients are combined (sample-weighted mean), the master
applies momentum SGD with whole-update non-finite rejection and every worker
continues from the new weights.  One process per GPU; at N=1 the master and
the single worker share GPU 0 and a round is one fused sm_100a kernel.

Prints ONE JSON line (rank 0).  `value` is device-timed (CUDA events on the
launching stream, inputs resident in HBM); `e2e` is the same metric through
the C ABI with HOST batches (H2D of each round's batch and D2H of its loss
inside the timed region).  The reference arm (`--impl reference`) runs the
reference's own CPU code (oracle/_ref: nn.cpp/optim.cpp/transport.cpp + the
SPEC roles over InprocHub) on this box's host cores.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ARCH = "lstm(5,20,10),softmax(20,3)"
FLOP_PER_SAMPLE = 102_760   # fwd 36,920 + bwd 65,840
SGD_BYTES_PER_PARAM = 20    # read w, v, g; write w, v (fp32)
WIDE_P = 16_881_699         # SURVEY §8 wide variant parameter count
WIDE_ARCH = "lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3)"
METRIC = "train samples/sec at 1/2/4/8 B200 (sync Downpour); % of roofline"
UNIT = "samples/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled over the clock window: a
    busy pre-roll of the same kernel (so the GPU is at its load clocks when
    the timed region starts — an idle GPU drops to 120 MHz within ~1 s) plus
    the timed region itself.  nvidia-smi's 20 ms period is longer than a
    20-round timed region (~0.3 ms), so `bracket` adds NVML reads taken
    immediately before and after the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.bracket = []
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self.nvml = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def started(self):
        """nvidia-smi delivered its first row (it needs ~0.1-1 s)."""
        return self.proc is None or bool(self.rows)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def mark(self, tag):
        """NVML clock read (bracket of the timed region)."""
        if self.nvml is None:
            return
        try:
            nv, h = self.nvml
            self.bracket.append({"at": tag, "sm_mhz": nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                 "reasons": int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))})
        except Exception:
            pass

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 7:
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        # NVML reason bits: 0x8 hw_slowdown, 0x20 sw_thermal, 0x40 hw_thermal, 0x4 sw_power_cap
        for b in self.bracket:
            for bit, nm in ((0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"),
                            (0x20, "sw_thermal_slowdown"), (0x4, "sw_power_cap")):
                if b["reasons"] & bit:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "window": "busy pre-roll of the same kernel + timed region",
                "bracket": self.bracket}


def preroll(run_chunk, ctx, clk, min_s=0.25):
    """Keep the GPU busy with the bench's own kernel (untimed) until the
    clock sampler runs and the clocks are at their load level."""
    t0 = time.time()
    while time.time() - t0 < min_s or not clk.started():
        run_chunk()
        ctx.sync()
        if time.time() - t0 > 10.0:
            break


def under_profiler() -> bool:
    """ncu/nsys inject into the process and serialise kernels — the gate
    kernel and the resident round service (kernels waiting on other work)
    cannot run under them, so the gate is skipped and the resident
    measurements too (paper_1712_05878_b200/_lib.py PROFILER_ENV)."""
    from paper_1712_05878_b200 import _lib
    return _lib.under_profiler()


def dist_env():
    # GHC_BENCH_DEVICE pins every rank to one device (validation of the N > 1
    # path with all ranks sharing one GPU under MPS, tools/gpurun_r2_mps_bench.sh)
    dev = os.environ.get("GHC_BENCH_DEVICE")
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(dev) if dev is not None else int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------------------
# reference arm: the reference's own CPU code (oracle/_ref)
# --------------------------------------------------------------------------
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    ncores = os.cpu_count() or 1
    W = args.ref_workers if args.ref_workers > 0 else max(1, min(ncores - 1, 96))
    spec = O.data_spec(96, 9500)
    cfg = O.train_cfg(n_workers=W, batch_size=args.batch, epochs=1000)
    # each step = one sync round of W workers × B samples; bounded sample
    steps = max(1, min(args.steps, args.ref_rounds))
    warm = max(3, min(args.warmup, 10))  # W ≥ 3, bounded: each round is ~0.1 s of CPU
    sec, n = O.ref_bench_sync(ARCH, spec, cfg, warm, steps)
    value = n / sec
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * sec / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "sync Downpour, lstm(5,20,10)+softmax(20,3), B=1000/worker",
                   "workers": W, "batch_per_worker": args.batch, "dataset_files": 96,
                   "samples_per_file": 9500},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": W + 1, "kind": "reference",
                         "sample": f"{steps} timed sync rounds × {W} worker threads × "
                                   f"B={args.batch} (reference nn/optim over InprocHub, "
                                   f"1 master thread + {W} worker threads on {ncores} cores)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args):
    """oracle/_ref sync Downpour at the bench's own config (W=1, B=1000)."""
    try:
        from oracle import oracle as O
        spec = O.data_spec(96, 9500)
        cfg = O.train_cfg(n_workers=1, batch_size=args.batch, epochs=1000)
        sec, n = O.ref_bench_sync(ARCH, spec, cfg, 2, args.cpu_rounds)
        return {"value": n / sec, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"{args.cpu_rounds} sync rounds, 1 worker × B={args.batch} "
                          "(reference nn.cpp/optim.cpp over InprocHub; 1 busy core + idle "
                          "master thread)"}
    except Exception as e:  # reported, never fatal
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_ours(args):
    import paper_1712_05878_b200 as g
    rank, world, local = dist_env()
    if world > 1:
        return run_ours_dist(args, rank, world, local)
    ctx = g.Context(local)
    arch = g.Architecture(ctx, ARCH)
    B = args.batch

    # dataset: DatasetSpec{96 files × 9500, T=10, D=5, K=3, δ=5, seed 1234}
    # (SURVEY §8(d)); the single worker's shard = all 96 files = 182 MB f32,
    # larger than the 126 MB L2, and every round gathers a fresh shuffled batch.
    t0 = time.time()
    spec = g.data_spec(96, 9500)
    x, y = g.generate(spec)
    total_rounds = args.warmup + args.steps
    per_epoch = x.shape[0] // B
    epochs = (total_rounds + per_epoch - 1) // per_epoch
    stream = []
    for e in range(epochs):
        idx = g.epoch_indices(spec, 1, 0, e, 99)
        stream.extend(idx[i:i + B] for i in range(0, per_epoch * B, B))
    idx = np.concatenate(stream[:total_rounds]).astype(np.int32)
    # packed rows (x | label | pad: 256-B rows = 2 whole 128-B lines per
    # gathered sample, ghc_dataset_pack), the labels argument is then None
    dx = g.pack_dataset(ctx, ctx.upload(x), ctx.upload(y))
    dy = None
    di = ctx.upload(idx)
    setup_s = time.time() - t0

    w0 = g.init_weights(arch, 7)
    m = g.Master(arch, w0, 0.01, 0.9)
    loss = ctx.array(total_rounds)
    mpre = g.Master(arch, w0, 0.01, 0.9)  # pre-roll on its own master: the timed one is untouched
    m.sync_rounds(dx, dy, di, B, B, args.warmup, loss_out=loss)  # W warm-up rounds (untimed)
    with ClockSampler(local) as clk:
        preroll(lambda: mpre.sync_rounds(dx, dy, di, B, B, min(2000, total_rounds)), ctx, clk)
        ctx.sync()
        launches0 = ctx.launches
        clk.mark("start")
        # ---- headline: the K rounds as ONE persistent launch
        # (ghc_master_sync_rounds), CUDA events on the launching stream; the
        # launch is queued behind a gate kernel (ghc_stream_hold, nvbench's
        # blocking kernel) so the host's call is not inside — the device-side
        # launch, prologue and teardown are
        gate = not args.no_resident  # (no gate under a profiler either)
        if gate:
            ctx.hold()
        ctx.timer_start()
        m.sync_rounds(dx, dy, di, B, B, args.steps, loss_out=loss, idx_offset=args.warmup * B,
                      loss_offset=args.warmup)
        if gate:
            ctx.release()
        ms = ctx.timer_stop()
        ctx.sync()
        clk.mark("stop")
        launches = ctx.launches - launches0
        # ---- the same K rounds through the resident round service
        # (ghc_resident_*: kernel launched once, one stream-doorbell command)
        ms_res = None
        if not args.no_resident:
            mr = g.Master(arch, w0, 0.01, 0.9)
            res = g.Resident(mr, B, idle_seconds=30.0)
            res.submit_stream(dx, dy, di, B, args.warmup)
            ctx.sync()
            ctx.hold()
            ctx.timer_start()
            res.submit_stream(dx, dy, di, B, args.steps, idx_offset=args.warmup * B)
            ctx.release()
            ms_res = ctx.timer_stop()
            res.check()
            res.stop()
            del mr
    del mpre
    _, _, version, rejected = m.read()
    losses = loss.numpy() / B
    chunk = args.steps

    # ---- kernel-level: one round per launch, CUDA events per launch ----
    per_launch_ms = []
    for k in range(min(args.steps, 200)):
        ctx.timer_start()
        m.sync_rounds(dx, dy, di, B, B, 1, idx_offset=(k % total_rounds) * B)
        per_launch_ms.append(ctx.timer_stop())
    per_launch_ms.sort()
    one_round_ms = statistics.median(per_launch_ms)

    # ---- e2e: host batches through the C ABI, H2D + round + D2H per step ----
    e2e = run_e2e(args, g, ctx, arch, x, y, idx)

    # ---- update path on the wide-variant parameter count (HBM roofline) ----
    upd = update_roofline(args, g, ctx)
    line = result_line(args, world, ms, one_round_ms, chunk, e2e, upd, launches, clk.summary(),
                       version, rejected, losses, setup_s, arch.kernel_name,
                       cpu_baseline(args) if not args.no_cpu else None)
    line["timing"] = {"method": "CUDA events on the launching stream around ONE persistent "
                                "launch of the K rounds (device-side launch, prologue and teardown "
                                "inside); the launch is queued behind a gate kernel so the host's "
                                "call is not",
                      "resident": {"ms_per_step": ms_res / args.steps if ms_res else None,
                                   "value": B * args.steps / (ms_res / 1e3) if ms_res else None,
                                   "path": "the same K rounds through the resident round service "
                                           "(ghc_resident_*): kernel launched once, one "
                                           "stream-doorbell command (submit+wait kernel → rounds → "
                                           "completion) inside the events"}}
    print(json.dumps(line), flush=True)
    return 0


# ncu --set full of one 200-round launch of lstm_round_kernel<5,20,10,3,4> on the
# packed dataset (profiles/r02_ncu_round_raw.csv): dram__bytes_read.sum 53.46 MB
# + dram__bytes_write.sum 0.52 MB → per round.  Algorithmic: the gathered batch
# + its indices, 1000 × (50 + 1 + 1) × 4 B = 208 KB; the packed 256-B rows are
# two whole 128-B lines each (the unpacked 200-B rows + separate labels cost
# 324.7 KB per round, profiles/r01_ncu_full_round_final_r1_raw.csv).
TRAFFIC_PER_ROUND = (53.456896e6 + 0.518912e6) / 200
TRAFFIC_SOURCE = ("ncu --set full, 200-round launch on packed rows (profiles/r02_ncu_round_raw.csv): "
                  "dram read+write / 200; traffic = per round × timed rounds")


# Latency/throughput roofline of the fused round (DESIGN.md §4 "latency
# roofline"): per phase the larger of the dependent-chain latency and the
# pipe-throughput bound, from the measured per-SM costs of tools/sm_micro.cu
# (profiles/r01_sm_micro.txt: dependent FFMA/FFMA2 4.9 cycles, EX2 17, SHFL
# 24, LDS 35, STS→syncwarp→LDS 34; broadcast LDS.128 2.79 SM-cycles and FFMA
# 1.24 SMSP-cycles per warp-instruction at 8 warps/SM) at 1965 MHz, and the
# measured L2 / DSMEM hop latencies of the exchange.
LATENCY_MODEL_US = {
    "forward": 1.15,        # 10 × (LDS h + 10-deep FFMA2 chain + σ/tanh MUFU chain + SHFL + cell) ≈ 225 cyc
    "softmax": 0.15,        # 3 butterfly sums + exp/log
    "bptt": 2.27,           # smem-throughput bound: 8 warps × 20 broadcast LDS.128 × 2.79 SM-cyc × 10 steps
    "weight_grads": 1.26,   # issue bound: 1000 FFMA per warp, 2 warps per SMSP × 1.24 cyc
    "exchange": 2.10,       # DSMEM push 0.3 + 2 × L2 store→poll 0.7 + SGD 0.1 + DSMEM push 0.3
}


def result_line(args, world, ms, one_round_ms, chunk, e2e, upd, launches, clocks, version,
                rejected, losses, setup_s, kernel, cpu):
    pk, pk_kind = peaks()
    B = args.batch
    steps_s = ms / 1e3
    value = world * B * args.steps / steps_s
    flops_per_round = B * FLOP_PER_SAMPLE  # per rank (GPU): one kernel launch each
    achieved_tflops = flops_per_round * args.steps / steps_s / 1e12
    tensor_peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) / 2.0  # TF32 ≈ ½ bf16
    fp32_peak = 148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SPEC generator, 96 files x 9500 samples per worker, delta=5)",
        "config": {"workload": "c2 sync Downpour, 1 master + 1 worker per GPU, "
                               "lstm(5,20,10)+softmax(20,3), B=1000/worker",
                   "global_batch": B * world, "seq_len": 10, "parallelism": f"dp{world}",
                   "rounds_per_launch": chunk,
                   "exchange": "in-kernel (DSMEM + L2)" if world == 1 else
                               ("in-kernel over NVLink peer memory (ghc_p2p)" if args.exchange == "p2p"
                                else f"NCCL {args.exchange} over NVLink"),
                   "l2": "inputs larger than L2: 182 MB shard/GPU > 126 MB L2, fresh "
                         "shuffled batch gathered every round"},
        # per GPU = per launch of the dominant kernel (each rank runs one)
        "roofline": {"bound": "tensor", "achieved": achieved_tflops,
                     "peak": tensor_peak, "unit": "TFLOP/s",
                     "frac": achieved_tflops / tensor_peak,
                     "traffic": args.traffic * args.steps if args.traffic else None,
                     "traffic_per_round_bytes": args.traffic,
                     "algorithmic_bytes_per_round": B * (10 * 5 + 1 + 1) * 4,
                     "traffic_source": TRAFFIC_SOURCE,
                     "kernel": kernel + " (fused fwd+bwd+reduce+SGD)",
                     "peak_kind": f"{pk_kind} bf16 sustained / 2 (TF32) per GPU",
                     "fp32_core": {"peak": fp32_peak,
                                   "frac": achieved_tflops / fp32_peak,
                                   "note": "the kernel is FFMA/MUFU/sync-bound by design "
                                           "(DESIGN.md §4)"},
                     "one_round_launch_ms": one_round_ms,
                     "latency": {"ideal_us_per_round": sum(LATENCY_MODEL_US.values()),
                                 "achieved_us_per_round": 1e3 * ms / args.steps,
                                 "frac": sum(LATENCY_MODEL_US.values()) / (1e3 * ms / args.steps),
                                 "phases_us": LATENCY_MODEL_US,
                                 "note": "the round is latency/smem-throughput bound, not FLOP "
                                         "bound: per-phase critical path or pipe-throughput "
                                         "bound from measured per-SM costs (DESIGN.md §4)"}},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "update_kernel": upd,
        "gpu_launches": launches,
        "clocks": clocks,
        "training": {"version": version, "rejected": rejected,
                     "loss_first": float(losses[0]), "loss_last": float(losses[-1])},
        "setup_s": setup_s,
    }


def run_ours_dist(args, rank, world, local):
    """N > 1: one worker per GPU.  Default exchange: the fused NVLink path
    (ghc_p2p_sync_rounds — the round kernels reduce through peer memory);
    --exchange reduce_bcast / allreduce: NCCL per round (ghc_dist_sync_rounds)."""
    import torch
    import torch.distributed as tdist

    import paper_1712_05878_b200 as g
    from paper_1712_05878_b200 import dist as gd
    tdist.init_process_group("gloo")
    ctx = g.Context(local)
    arch = g.Architecture(ctx, ARCH)
    B = args.batch
    p2p = args.exchange == "p2p"
    if p2p:
        try:
            ex = gd.P2PExchange(arch, rank, world, dist=tdist)
        except gd.P2PUnavailable as e:  # raised on every rank alike
            print(f"[bench] fused NVLink exchange unavailable ({e}); using NCCL reduce/broadcast",
                  file=sys.stderr)
            p2p = False
            args.exchange = "reduce_bcast"
    if not p2p:
        uid = gd.rendezvous(tdist, rank, gd.nccl_unique_id)
        comm = gd.Comm(ctx, uid, rank, world)
        exchange = gd.ALLREDUCE if args.exchange == "allreduce" else gd.REDUCE_BCAST
    t0 = time.time()
    spec = g.data_spec(96 * world, 9500)  # weak scaling: 96 files (182 MB) per worker
    total_rounds = args.warmup + args.steps
    per_epoch = 96 * 9500 // B
    epochs = (total_rounds + per_epoch - 1) // per_epoch
    plan = gd.plan_worker(spec, world, rank, B, epochs, 99)
    counts = gd.round_counts(spec, world, B, epochs, 99)[:total_rounds]
    x, y = g.generate(spec, plan.first_file, plan.n_files)
    if p2p:  # packed rows (x | label | pad to 256 B) for the fused exchange's round kernel
        dx, dy = g.pack_dataset(ctx, ctx.upload(x), ctx.upload(y)), None
    else:
        dx, dy = ctx.upload(x), ctx.upload(y)
    di = ctx.upload(plan.idx_local[: total_rounds * B])
    dc = ctx.upload(np.ascontiguousarray(counts, np.int32))
    setup_s = time.time() - t0
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    loss = ctx.array(total_rounds)
    state = {"m": m}

    def rounds(r0, n, loss_offset, lbuf=None):
        m = state["m"]
        lbuf = loss if lbuf is None else lbuf
        if p2p:
            ex.sync_rounds(m, dx, dy, di, B, 0, dc, B, n, loss_out=lbuf, idx_offset=r0 * B,
                           counts_offset=r0 * world, loss_offset=loss_offset)
        else:
            gd.dist_sync_rounds(m, comm, exchange, dx, dy, di, B, counts[r0:r0 + n], n,
                                lbuf, idx_offset=r0 * B)

    rounds(0, args.warmup, 0)
    ctx.sync()
    tdist.barrier()
    with ClockSampler(local) as clk:
        # busy pre-roll (untimed, same number of calls on every rank: the
        # fused exchange pairs the ranks' rounds) on a scratch master
        state["m"] = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
        scratch_loss = ctx.array(total_rounds)  # the scratch master's losses stay out of the report
        for _ in range(args.preroll_calls):
            rounds(0, min(total_rounds, 2000), 0, scratch_loss)
        ctx.sync()
        state["m"] = m
        launches0 = ctx.launches
        tdist.barrier()
        ctx.sync()
        tdist.barrier()
        clk.mark("start")
        gate = not under_profiler()
        if gate:
            ctx.hold()  # queue the timed launches behind a gate (device time only)
        # device-side barrier of the ranks right before the start event: the
        # processes' gates open tens of µs apart after the host barrier,
        # which the max over ranks would otherwise count
        if p2p:
            ex.device_barrier()
        else:
            comm.device_barrier()
        ctx.timer_start()
        rounds(args.warmup, args.steps, args.warmup)
        if gate:
            ctx.release()
        ms_local = ctx.timer_stop()
        ctx.sync()
        clk.mark("stop")
        tdist.barrier()
    t = torch.tensor([ms_local], dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    launches = ctx.launches - launches0
    _, _, version, rejected = m.read()
    losses = loss.numpy() / (B * world)
    e2e = None
    if p2p:
        e2e = run_e2e_dist(args, g, gd, tdist, ctx, arch, ex, x, y, plan, dc, rank, world)
    if rank == 0:
        line = result_line(args, world, ms, None, args.steps, e2e, None, launches, clk.summary(),
                           version, rejected, losses, setup_s, arch.kernel_name, None)
        print(json.dumps(line), flush=True)
    tdist.barrier()
    if p2p:
        ex.close()
    tdist.destroy_process_group()
    return 0


def run_e2e_dist(args, g, gd, tdist, ctx, arch, ex, x, y, plan, dc, rank, world):
    """e2e at N GPUs through the public API: every rank streams its K batches
    from pinned host memory (zero-copy, as run_e2e) through ONE
    ghc_p2p_sync_rounds call; time = max over ranks."""
    import torch
    B = args.batch
    K = min(args.steps, args.e2e_steps)
    width = x.shape[1]
    sel = plan.idx_local[: K * B]
    xs = g.pack_rows(x[sel], y[sel])
    hx = ctx.host_array(xs.shape)
    hy = None
    hl = ctx.host_array(K)
    hx.np[:] = xs
    hl.np[:] = np.nan
    m = g.Master(arch, g.init_weights(arch, 7), 0.01, 0.9)
    ctx.sync()
    tdist.barrier()
    ex.device_barrier()  # align the ranks' start events on the device (no host skew)
    ctx.timer_start()
    ex.sync_rounds(m, hx, hy, None, B, 0, dc, B, K, loss_out=hl)
    ms_local = ctx.timer_stop()
    ctx.sync()
    tdist.barrier()
    t = torch.tensor([ms_local], dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    ok = bool(np.isfinite(hl.np).all())
    for a in (hx, hl):
        a.free()
    return {"value": world * B * K / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": world * B * (width + 1) * 4, "d2h_bytes_per_step": world * 4,
            "steps": K, "ms_per_step": ms / K, "losses_finite": ok,
            "path": "per rank: ghc_p2p_sync_rounds over K host batches (pinned, zero-copy "
                    "prefetch one round ahead, losses stored to host memory); max over ranks"}


def run_e2e(args, g, ctx, arch, x, y, idx):
    """Same metric through the public API with the data on the HOST:

    * host_dataset (the headline ``e2e``): the worker's whole 182 MB shard,
      its labels and the shuffled index stream live in pinned host memory
      (HostArray), like the reference's in-memory dataset; ONE
      ghc_master_sync_rounds call trains K rounds and every round the
      persistent kernel gathers its freshly shuffled batch rows straight
      from host memory over PCIe (cp.async, one round ahead) and stores the
      round's loss to host memory.  The batch assembly the reference arm does
      per round (oracle/ref_roles.cpp:139-143) is inside the timed region;
      CUDA events around the call (host launch call included).
    * host_dataset_resident: the same through the resident round service
      (ghc_resident_submit + ghc_resident_wait, host doorbell), host clock.
    * pregathered: the K batches already gathered contiguously in pinned
      host memory (the gather done before timing), one call.
    * per_call: one batch per call — ghc_resident_submit(1 round) +
      ghc_resident_wait per batch (loss back in host memory when the call
      returns), host clock; per_call_launch: one ghc_master_sync_rounds
      launch per batch, calls queued on one stream, CUDA events."""
    B = args.batch
    K = min(args.steps, args.e2e_steps)
    width = x.shape[1]
    w0 = g.init_weights(arch, 7)

    def launched(xs, ys, ix, stride, rounds, loss_out):
        m = g.Master(arch, w0, 0.01, 0.9)
        m.sync_rounds(xs, ys, ix, stride, B, min(3, rounds), loss_out=loss_out)  # warm-up
        ctx.sync()
        # busy pre-roll (untimed, same kernel and data): the host-side packing
        # above leaves the GPU idle long enough to drop its clocks
        t0 = time.time()
        while time.time() - t0 < 0.25:
            m.sync_rounds(xs, ys, ix, stride, B, rounds, loss_out=loss_out)
            ctx.sync()
        m = g.Master(arch, w0, 0.01, 0.9)
        loss_out.np[:] = np.nan
        ctx.sync()
        ctx.timer_start()
        m.sync_rounds(xs, ys, ix, stride, B, rounds, loss_out=loss_out)
        t = ctx.timer_stop() / 1e3
        ctx.sync()
        return t

    def served(xs, ys, ix, stride, rounds, loss_out):
        m = g.Master(arch, w0, 0.01, 0.9)
        res = g.Resident(m, B)
        scratch = ctx.host_array(3)
        res.wait(res.submit(xs, ys, ix, stride, 3, loss_out=scratch))  # warm-up command
        loss_out.np[:] = np.nan
        t0 = time.perf_counter()
        res.wait(res.submit(xs, ys, ix, stride, rounds, loss_out=loss_out))
        dt = time.perf_counter() - t0
        res.stop()
        scratch.free()
        return dt

    # ---- host_dataset (packed rows: x | label | pad, 256 B) ----
    xp = g.pack_rows(x, y)
    hX = ctx.host_array(xp.shape)
    hY = None
    hI = ctx.host_array(K * B, np.int32)
    hl = ctx.host_array(K)
    hX.np[:] = xp
    hI.np[:] = idx[: K * B]
    del xp
    dt = launched(hX, hY, hI, B, K, hl)
    out = {"value": B * K / dt, "unit": UNIT,
           "h2d_bytes_per_step": B * (width * 4 + 4 + 4), "d2h_bytes_per_step": 4,
           "h2d_bytes_moved_per_step": B * (64 * 4 + 4),
           "steps": K, "ms_per_step": 1e3 * dt / K, "losses_finite": bool(np.isfinite(hl.np).all()),
           "path": "ghc_master_sync_rounds with the dataset (182 MB), labels and shuffled index "
                   "stream in pinned host memory: each round's batch is gathered by the kernel "
                   "from host memory over PCIe (one round ahead), its loss stored to host memory"}
    if not args.no_resident:
        dtr = served(hX, hY, hI, B, K, hl)
        out["host_dataset_resident"] = {"value": B * K / dtr, "ms_per_step": 1e3 * dtr / K,
                                        "losses_finite": bool(np.isfinite(hl.np).all()),
                                        "clock": "host perf_counter around submit + wait",
                                        "path": "the same through ghc_resident_submit/wait (host "
                                                "doorbell)"}
    for a in (hX, hI):
        a.free()

    # ---- pregathered ----
    sel = idx[: K * B]
    xs = g.pack_rows(x[sel], y[sel])
    hx = ctx.host_array(xs.shape)
    hy = None
    hx.np[:] = xs
    dtp = launched(hx, hy, None, B, K, hl)
    out["pregathered"] = {"value": B * K / dtp, "steps": K, "ms_per_step": 1e3 * dtp / K,
                          "losses_finite": bool(np.isfinite(hl.np).all()),
                          "path": "K batches pre-gathered contiguously in pinned host memory (gather "
                                  "outside the timed region); one call streams them zero-copy"}

    # ---- per_call: one batch per call ----
    Kc = min(K, 200)
    if not args.no_resident:
        m = g.Master(arch, w0, 0.01, 0.9)
        res = g.Resident(m, B)
        hl.np[:] = np.nan
        for k in range(3):
            res.wait(res.submit(hx.sub(k * B), None, None, 0, 1, loss_out=hl.sub(k)))
        t0 = time.perf_counter()
        for k in range(Kc):
            res.wait(res.submit(hx.sub(k * B), None, None, 0, 1, loss_out=hl.sub(k)))
        dtc = time.perf_counter() - t0
        # queued: up to 3 batches in flight — batch k+2 submitted before
        # waiting for batch k (the kernel fetches the next command's batch
        # during the current command's round when it is already queued)
        hl.np[:] = np.nan
        t0 = time.perf_counter()
        seqs = []
        for k in range(Kc):
            seqs.append(res.submit(hx.sub(k * B), None, None, 0, 1, loss_out=hl.sub(k)))
            if k >= 2:
                res.wait(seqs[k - 2])
        res.wait(seqs[-1])
        dtq = time.perf_counter() - t0
        # the same loops in C++ over the C ABI (a reference-side caller; no
        # interpreter between the calls)
        import ctypes as C
        us = {}
        for depth in (1, 3, 6):
            u = C.c_double()
            g.gradhub.check(ctx.lib.ghc_resident_bench_calls(res.h, hx.ptr, B * hx.shape[1], None, 0, Kc,
                                                             depth, hl.ptr, C.byref(u)), "bench_calls")
            us[depth] = u.value
        res.stop()
        out["per_call_cxx"] = {"value": B / (us[6] * 1e-6), "ms_per_step": us[6] / 1e3, "depth": 6,
                               "depth3_ms_per_step": us[3] / 1e3,
                               "synchronous_ms_per_step": us[1] / 1e3,
                               "losses_finite": bool(np.isfinite(hl.np[:Kc]).all()),
                               "path": "ghc_resident_bench_calls: a C++ loop over ghc_resident_submit "
                                       "(1 round, batch zero-copy from pinned host memory) + "
                                       "ghc_resident_wait, up to 6 batches in flight (a host batch "
                                       "is fetched over PCIe a whole round ahead once its command is "
                                       "queued two commands early; depth 3 and synchronous depth 1 "
                                       "also reported); host wall clock"}
        out["per_call"] = {"value": B * Kc / dtq, "steps": Kc, "ms_per_step": 1e3 * dtq / Kc,
                           "losses_finite": bool(np.isfinite(hl.np[:Kc]).all()),
                           "clock": "host perf_counter",
                           "path": "per batch: ghc_resident_submit(1 round, batch zero-copy from "
                                   "pinned host memory) + ghc_resident_wait, up to 3 batches in "
                                   "flight (losses land in host memory)",
                           "synchronous": {"ms_per_step": 1e3 * dtc / Kc,
                                           "path": "submit + wait per batch, nothing queued"}}
    m = g.Master(arch, w0, 0.01, 0.9)
    for k in range(3):
        m.sync_rounds(hx.sub(k * B), None, None, 0, B, 1, loss_out=hl.sub(k))
    ctx.sync()
    ctx.timer_start()
    for k in range(Kc):
        m.sync_rounds(hx.sub(k * B), None, None, 0, B, 1, loss_out=hl.sub(k))
    msl = ctx.timer_stop()
    ctx.sync()
    out["per_call_launch"] = {"value": B * Kc / (msl / 1e3), "steps": Kc, "ms_per_step": msl / Kc,
                              "path": "one ghc_master_sync_rounds(1 round) launch per batch, queued "
                                      "on one stream (CUDA events)"}
    for a in (hx, hl):
        a.free()
    return out


L2_NOTE = ("steady-state streaming: NSET back-to-back launches over distinct buffer sets "
           "(8 × the working set ≫ the 126 MB L2: no reuse between launches, and every launch "
           "pays the write-back of its predecessor's dirty lines); time / NSET per launch")
NSET = 8


def update_roofline(args, g, ctx):
    """The master's update path (optim.cpp:39-65) at the wide variant's P,
    HBM roofline: ghc_master_apply (one pass into the other buffer,
    sgd_db_kernel — what a Downpour master runs per combined gradient) and
    the in-place ghc_sgd_apply (finite check + update, sgd_apply_kernel)."""
    P = WIDE_P
    rng = np.random.default_rng(0)
    w0 = rng.normal(size=P).astype(np.float32)
    grs = [ctx.upload((rng.normal(size=P) * 1e-3).astype(np.float32)) for _ in range(NSET)]
    pk, kind = peaks()

    def timed(fns):
        times = []
        for it in range(8):
            ctx.sync()
            ctx.timer_start()
            for fn in fns:
                fn()
            t = ctx.timer_stop() / len(fns)
            if it >= 2:
                times.append(t)
        return statistics.median(times)

    arch = g.Architecture(ctx, WIDE_ARCH)
    assert arch.n_params == P
    ms = [g.Master(arch, w0, 0.01, 0.9) for _ in range(NSET)]
    t_db = timed([lambda m=m, gr=gr: m.apply(gr) for m, gr in zip(ms, grs)])
    del ms
    ws = [ctx.upload(w0) for _ in range(NSET)]
    vs = [ctx.upload(np.zeros(P, np.float32)) for _ in range(NSET)]
    st = ctx.array(1, np.int32)
    t_ip = timed([lambda w=w, v=v, gr=gr: g.gradhub.check(ctx.lib.ghc_sgd_apply(
        ctx.h, w.ptr, v.ptr, gr.ptr, P, 0.01, 0.9, st.ptr, None)) for w, v, gr in zip(ws, vs, grs)])

    def row(kernel, t):
        gbs = SGD_BYTES_PER_PARAM * P / (t / 1e3) / 1e9
        return {"kernel": kernel, "P": P, "ms": t, "achieved_gbs": gbs, "peak_gbs": pk["hbm_gbs"],
                "frac": gbs / pk["hbm_gbs"], "bytes_per_param": SGD_BYTES_PER_PARAM,
                "peak_kind": kind, "l2": L2_NOTE}
    out = row("sgd_db_kernel", t_db)
    out["in_place"] = row("sgd_apply_kernel", t_ip)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1000)
    ap.add_argument("--chunk", type=int, default=0, help="rounds per persistent launch (0=all)")
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--cpu-rounds", type=int, default=120)
    ap.add_argument("--ref-rounds", type=int, default=40)
    ap.add_argument("--ref-workers", type=int, default=0,
                    help="reference arm worker threads (0: one per host core, minus the master)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-resident", action="store_true",
                    help="skip the resident-service measurements (automatic under ncu/nsys)")
    ap.add_argument("--preroll-calls", type=int, default=20,
                    help="N>1: untimed busy calls before the timed region (same on every rank)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "reduce_bcast", "allreduce"])
    ap.add_argument("--traffic", type=float, default=TRAFFIC_PER_ROUND,
                    help="dram bytes per round of the fused kernel from an ncu --set full capture")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if under_profiler():
        args.no_resident = True
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args.gpus)
    _, world, _ = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


def spawn(n):
    """`bench.py --gpus N` without a launcher: run this same command as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())

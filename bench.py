#!/usr/bin/env python3
"""Tree-attention decode benchmark (BASELINE.json metric: decode-attention
latency in us per decoded token at 1/2/4/8 B200, plus HBM GB/s).

Workload (default): Llama-3-8B attention shape -- 32 q / 8 kv heads, d 128,
bf16, 1,048,576-token KV cache sharded over the N GPUs (BASELINE.json
configs[2], the north-star target). A step is one decode of one new token:
K1+K2 on every rank's shard, allreduce(max), K3, allreduce(sum), K4.
Total work is fixed as N grows ("scaling": "strong").

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                  [--workload cfg1|cfg2|cfg3|cfg4] [--seq-len N] [--algo tree|ring]

Multi-GPU: launched by torchrun, one rank per GPU, NCCL. The timed region is
bracketed by a barrier + cuda synchronize on both sides; every step is timed
with CUDA events on the library's stream; the reported time is the max over
ranks. Inputs are generated on the device with the reference generator
(synthetic data, bit-exact with the CPU reference); the KV shard of every
rank exceeds L2 at the default workload, otherwise L2 is flushed between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (description, b, n_q, n_kv, seq_len, d, dtype)
    "cfg1": ("single-head decode, 64K-token KV, d=128, fp32 (configs[0])", 1, 1, 1, 65536, 128, "f32"),
    "cfg2": ("32-head MHA decode, batch 1, 256K tokens, bf16 (configs[1])", 1, 32, 32, 262144, 128, "bf16"),
    "cfg3": ("Llama-3-8B attention (32q/8kv GQA, d=128), 1M-token KV, bf16 (configs[2])", 1, 32, 8, 1048576, 128,
             "bf16"),
    "cfg4": ("batch 16 decode, 128K tokens per sequence, GQA 8:1 (64q/8kv), bf16 (configs[3])", 16, 64, 8, 131072,
             128, "bf16"),
}
METRIC = "decode-attn latency (µs/token) vs seq len at 1/2/4/8 B200; HBM GB/s"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3")
    ap.add_argument("--seq-len", type=int, default=None)
    ap.add_argument("--algo", choices=["tree", "ring"], default="tree")
    ap.add_argument("--combine", choices=["nccl", "p2p", "nccl_device"], default="p2p",
                    help="tree exchange (N > 1): one-shot NVLink exchange (default; falls back to nccl "
                         "if CUDA IPC is unavailable on any rank), two NCCL allreduces (paper-literal), or "
                         "the same two allreduces inside one kernel through NCCL's device API")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-heads", type=int, default=None)
    ap.add_argument("--phases", action="store_true", help="add a per-phase breakdown (phases_us)")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed output")
    ap.add_argument("--no-compare", action="store_true",
                    help="N > 1: skip the ring pass-KV and paper-literal NCCL comparison records")
    ap.add_argument("--compare-steps", type=int, default=10)
    ap.add_argument("--dynamic", action="store_true",
                    help="dynamic tile pool (TD_DYNAMIC; the default static split is bitwise reproducible)")
    return ap.parse_args()


def interconnect(args, world, b, n_q, n_kv, n, d, esz, ms):
    """NVLink payload per rank per step and its rate over the step (a lower bound
    on the bus rate: the transfers overlap compute). Ring: the p-1 KV chunks each
    rank receives; tree: the exchange (LL words of [out | lse] to every peer, or
    the payload of NCCL's max and sum allreduces)."""
    if world == 1:
        return None
    rows = b * n_q
    if args.algo == "ring":
        per_tok = b * n_kv * d * esz * 2
        base, extra = divmod(n, world)
        chunk = [base + (1 if i < extra else 0) for i in range(world)]
        nbytes = sum(chunk) - chunk[0]  # every rank receives all chunks but its own (max over ranks ~ this)
        nbytes *= per_tok
        what = "ring pass-KV: KV chunks received per rank (NCCL send/recv)"
    elif args.combine == "p2p":
        nbytes = (world - 1) * rows * (d + 1) * 8
        what = "one-shot exchange: LL words (value, epoch) of [out | lse] pushed to every peer"
    elif args.combine == "nccl_device":
        nbytes = (world - 1) * rows * (d + 2) * 8
        what = "NCCL device API: LL words of lse, then of [n | d], stored into every rank's symmetric window"
    else:
        nbytes = rows * 4 + rows * (d + 1) * 4
        what = "NCCL allreduce(max) of lse + allreduce(sum) of [n | d] (payload)"
    return {"kind": "nvlink", "bytes_per_rank_per_step": nbytes, "gbs": nbytes / (ms * 1e-3) / 1e9, "what": what}


def read_ceiling(nbytes):
    """The measured ceiling of a plain streaming-read kernel at the nearest
    working-set size (scripts/read_probe.cu, profiles/r2_read_ceiling.jsonl):
    MEASURED_PEAKS.json's HBM figure is a read+write copy, which a read-only
    stream exceeds at large sizes and cannot reach at small ones (ramp)."""
    path = os.path.join(ROOT, "profiles", "r2_read_ceiling.jsonl")
    try:
        rows = [json.loads(x) for x in open(path) if x.startswith("{")]
    except OSError:
        return None
    if not rows:
        return None
    mb = nbytes / 1e6
    near = min(rows, key=lambda r: abs(math.log(r["mb"] / mb)))
    return {"gbs": near["gbs"], "at_mb": near["mb"], "how": near["how"], "source": near["source"]}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(workload, algo, shard_tokens):
    """dram bytes per K1 launch from the committed ncu summary (keyed by the
    shard's tokens per (batch, kv-head) row), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s.get(f"{workload}/{algo}/t{shard_tokens}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[1]) for s in self.samples if len(s) > 2 and s[1].replace(".", "").isdigit())
        mx = max((float(s[2]) for s in self.samples if len(s) > 2 and s[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 9 for i in range(4)
                          if s[5 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def barrier(world):
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def align_streams(world, stream):
    """After a host barrier the ranks' GPUs start their queues up to hundreds of
    us apart, and the first exchange of the timed loop would absorb that skew.
    A one-element NCCL allreduce, followed on the library stream by a
    device-side wait (no host sync), releases every rank's first step within
    microseconds of each other."""
    if world == 1:
        return
    import torch
    import torch.distributed as dist
    t = torch.ones(1, device="cuda")
    dist.all_reduce(t)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream())
    stream.wait_event(ev)


def bench_config(args, wl, world, combine, flush):
    """The config dict of a bench line (both arms: the driver matches them key by key)."""
    desc, b, n_q, n_kv, n, d, dt = wl
    n = args.seq_len or n
    return {"workload": args.workload, "desc": desc, "seq_len": n, "batch": b, "q_heads": n_q,
            "kv_heads": n_kv, "head_dim": d, "shards": world, "shard_tokens": math.ceil(n / world),
            "algo": args.algo, "combine": combine, "scale": args.scale,
            "nccl_algo": os.environ.get("NCCL_ALGO", "auto") if world > 1 else None,
            "l2": "flushed between steps (read-only sweep of 256 MB, timed apart and subtracted)" if flush
            else "inputs larger than L2 (KV shard > 4x126 MB)",
            "parallelism": f"sp{world} (sequence-sharded KV)",
            "deterministic": not getattr(args, "dynamic", False)}


def parity_leg(args, wl, q_dev, out_dev, world):
    """THE CHECKER (rank 0, after timing): the timed run's device output against
    the oracle -- the reference algorithm in Float64 on the same bf16 / f32
    inputs (oracle/full.py) -- on every row when b * n_q <= 64, else one query
    row per (batch, kv-head) pair, rotating through the group."""
    import numpy as np

    from oracle.full import full_decode, rel_err_rows
    from oracle.oracle import BF16, F32, Oracle
    _, b, n_q, n_kv, n, d, dt = wl
    n = args.seq_len or n
    t0 = time.time()
    orc = Oracle()
    seed = orc.mix64(0, n)
    dtc = BF16 if dt == "bf16" else F32
    qh = orc.seeded(orc.mix64(seed, 1), b * n_q * d, dtc).reshape(b, n_q, d)
    if not np.array_equal(q_dev.double().cpu().numpy(), qh):
        return {"max_rel_err": None, "ok": False, "note": "device query differs from the reference generator"}
    g = n_q // n_kv
    if b * n_q <= 64:
        rows = None
    else:
        rows = [(ib, kvh * g + (ib + kvh) % g) for ib in range(b) for kvh in range(n_kv)]
    want = full_decode(orc, qh, n_kv, n, orc.mix64(seed, 2), orc.mix64(seed, 3), dtc, args.scale, rows=rows)
    err = rel_err_rows(out_dev.double().cpu().numpy(), want)
    tol = 1e-3 if dt == "bf16" else 1e-5
    return {"max_rel_err": err, "tol": tol, "ok": bool(err <= tol), "rows_checked": len(want),
            "rows_total": b * n_q, "kv_rows_covered": len({(ib, h // g) for ib, h in want}),
            "oracle": "reference decode in Float64 on the same dtype-rounded inputs (oracle/treedec_oracle.c, "
                      "per (batch, kv-head) row, token-range partials + combine_partials)",
            "seconds": round(time.time() - t0, 1)}


# ---------------------------------------------------------------- CPU reference (oracle/_ref)
def reference_cpu(args, wl, n_gpus, sample_heads, nthreads, steps=1, warmup=0):
    """Times the reference's own tree_decode (compiled from /root/reference by
    oracle/Makefile into oracle/_ref) on a bounded sample: `sample_heads` query
    rows, all reading one kv head at the full sequence length (a row's cost
    does not depend on which kv head it reads, and one kv head keeps the f64
    inputs at 2 GB), p = n_gpus workers (parallel_workers when p > 1), the
    sampled rows spread over `nthreads` host threads; scaled linearly to all
    b * n_q rows. Inputs are built once (not timed, like shard_kv in
    BASELINE.md section 3); returns the per-step values."""
    from oracle.oracle import BF16, F32, HIER, Oracle, Reference
    _, b, n_q, n_kv, n, d, dt = wl
    n = args.seq_len or n
    orc, ref = Oracle(), Reference()
    dtc = BF16 if dt == "bf16" else F32
    seed = orc.mix64(0, n)
    rows = b * n_q
    sample_heads = max(1, min(sample_heads, rows))
    nthreads = max(1, min(nthreads, sample_heads))
    qh = orc.seeded(orc.mix64(seed, 1), sample_heads * d, dtc).reshape(1, sample_heads, d)
    k0 = orc.seeded(orc.mix64(seed, 2), n * d, dtc).reshape(1, 1, n, d)
    v0 = orc.seeded(orc.mix64(seed, 3), n * d, dtc).reshape(1, 1, n, d)
    vals = []
    with ref.prepare(qh, k0, v0, n_gpus, dtc) as pr:
        del k0, v0
        for i in range(warmup + steps):
            _, secs, _ = pr.decode(0, HIER, args.scale, parallel=n_gpus > 1, nthreads=nthreads)
            if i >= warmup:
                vals.append(secs / sample_heads * rows * 1e6)  # us per decode step (= per token of each sequence)
    cores = nthreads * (n_gpus if n_gpus > 1 else 1)
    return vals, {
        "sample": f"{sample_heads} query row(s) over one kv head at N={n}, p={n_gpus} worker(s), {nthreads} row "
                  f"thread(s); scaled x{rows / sample_heads:g} to b*n_q={rows} rows; inputs built once (untimed)",
        "cores": cores,
    }


def run_reference_arm(args, wl, world, rank):
    if rank != 0:
        return
    nproc = os.cpu_count() or 1
    _, b, n_q, n_kv, n, d, dt = wl
    # every host thread: p = N workers per call (threads), sampled rows in parallel
    row_threads = max(1, min(b * n_q, nproc // max(1, args.gpus)))
    heads = row_threads
    t0 = time.time()
    vals, info = reference_cpu(args, wl, args.gpus, heads, row_threads, steps=args.steps, warmup=args.warmup)
    value = sum(vals) / len(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "µs/token", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value / 1000.0, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": dt, "data": "synthetic (reference generator)",
        "config": bench_config(args, wl, args.gpus, combine=(args.combine if args.gpus > 1 and args.algo == "tree"
                                                             else "none"),
                               flush=2 * b * n_kv * math.ceil((args.seq_len or n) / args.gpus) * d
                               * (2 if dt == "bf16" else 4) < 4 * L2_BYTES),
        "cpu_baseline": {"value": value, "unit": "µs/token", "cores": info["cores"], "kind": "reference",
                         "sample": info["sample"] + f"; host nproc={nproc}, {cpu_model()}"},
        "e2e": {"value": value, "unit": "µs/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.time() - t0, 1),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    wl = WORKLOADS[args.workload]
    desc, b, n_q, n_kv, n, d, dt = wl
    n = args.seq_len or n
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference_arm(args, wl, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch

    import paper_2408_04093_b200 as td
    from paper_2408_04093_b200 import _capi
    torch.cuda.set_device(local)
    dtype = td.DType.Bf16 if dt == "bf16" else td.DType.Float32
    esz = 2 if dt == "bf16" else 4

    def mix64(seed, c):  # numerics.cpp:30-35 (seeding convention only, bench.cpp:73)
        m = (1 << 64) - 1
        z = (seed + ((c + 1) * 0x9E3779B97F4A7C15)) & m
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)

    seed = mix64(0, n)
    if args.dynamic:
        td.set_deterministic(False)
    w = td.Worker.from_torch_distributed(local) if world > 1 else td.Worker(local)
    w.generate_kv(dtype, b, n_kv, n, d, mix64(seed, 2), mix64(seed, 3))
    start, shard_len, shard_bytes = w.kv_info()
    q = td.seeded_tensor([b, n_q, d], mix64(seed, 1), 1.0, dtype)
    out = torch.empty(b, n_q, d, dtype=torch.float32, device="cuda")
    stream_ptr = w.stream
    stream = torch.cuda.ExternalStream(stream_ptr)
    flush = shard_bytes < 4 * L2_BYTES
    # L2 flush by a read-only sweep of 256 MB (> 2 x L2): it leaves clean lines, so
    # the decode that follows pays no write-back of a flush's dirty lines
    scratch = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda") if flush else None
    flush_sink = torch.empty((), dtype=torch.float32, device="cuda") if flush else None

    def flush_l2():
        torch.sum(scratch, dim=0, out=flush_sink)
    decode = w.tree_decode_async if args.algo == "tree" else w.ring_decode_async
    flags_timed = _capi.TD_TIME_KERNELS
    base_flags = 0
    if args.combine == "p2p" and world > 1 and args.algo == "tree":
        import torch.distributed as dist
        ok = 1
        try:
            w.enable_p2p(b * n_q, d)
        except Exception as e:  # every rank must agree before the first exchange
            print(f"rank {rank}: P2P exchange unavailable ({e}); using the NCCL path", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            base_flags = _capi.TD_P2P
        else:
            args.combine = "nccl"
    elif args.combine == "nccl_device" and world > 1 and args.algo == "tree":
        base_flags = _capi.TD_NCCL_DEVICE

    def step(flags):
        decode(q.data_ptr(), n_q, out.data_ptr(), args.scale, flags | base_flags)

    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 3)):
        if flush:  # the flush's own first-use costs (lazy module load, workspace) stay out of the timed steps
            with torch.cuda.stream(stream):
                flush_l2()
        step(0)
    barrier(world)

    # ---- device-timed region: K steps back to back (a decode loop), one CUDA
    # event pair on the library stream around all of them (per-step events
    # would sit between one step's K2 and the next step's K1 and so undo the
    # programmatic launch that hides the kernel-to-kernel gap); with an L2 flush
    # the flush kernels are timed separately and subtracted
    w.reset_kernel_timer()
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fl = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # pass A: the step as a user runs it
        barrier(world)
        align_streams(world, stream)
        ev_a.record(stream)
        for i in range(args.steps):
            if flush:
                fl[i][0].record(stream)
                with torch.cuda.stream(stream):
                    flush_l2()
                fl[i][1].record(stream)
            step(0)
        ev_b.record(stream)
        barrier(world)
        # pass B: the same steps with CUDA events around the split-KV kernel (K1)
        # for the roofline (an event between K1 and K2 would serialise the PDL
        # launch, so it is kept out of pass A)
        align_streams(world, stream)
        for i in range(args.steps):
            if flush:
                with torch.cuda.stream(stream):
                    flush_l2()
            step(flags_timed)
        barrier(world)
    out_timed = out.clone()  # the timed run's output (checked against the oracle below)
    flush_ms = sum(a.elapsed_time(bb) for a, bb in fl) if flush else 0.0
    ms_local = (ev_a.elapsed_time(ev_b) - flush_ms) / args.steps
    k1_ms, k1_calls = w.kernel_time()
    kernels_per_step, kv_bytes_step, split_kernel = w.last_launch_stats()
    ms = max_over_ranks(ms_local, world)
    lib_bytes = max_over_ranks(float(w.memory_bytes()), world)
    free_b, total_b = torch.cuda.mem_get_info()
    used_max = max_over_ranks(float(total_b - free_b), world)
    k1_ms_max = max_over_ranks(k1_ms, world)

    # ---- end-to-end through the public API with host buffers (pinned)
    q_host = q.cpu().pin_memory()
    out_host = torch.empty(b, n_q, d, dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))
    barrier(world)
    e2e_times = []
    for i in range(e2e_steps):
        if flush:
            with torch.cuda.stream(stream):
                flush_l2()
            stream.synchronize()
        t0 = time.perf_counter()
        decode(q_host.data_ptr(), n_q, out_host.data_ptr(), args.scale, _capi.TD_HOST_IO | _capi.TD_PINNED_IO | base_flags)
        e2e_times.append(time.perf_counter() - t0)
    e2e_ms = max_over_ranks(1000.0 * sum(e2e_times) / len(e2e_times), world)
    # same result through the host path; the dynamic tile pool regroups the
    # split-KV sums from call to call (~1e-7 relative), so not bitwise
    ref_out = out.cpu()
    ok = float((out_host - ref_out).abs().max()) <= 1e-5 * float(ref_out.abs().max())

    # ---- per-phase breakdown (separate pass, not part of the timed number)
    phases = None
    if args.phases:
        barrier(world)
        w.reset_kernel_timer()
        align_streams(world, stream)
        for _ in range(max(3, min(args.steps, 20))):
            step(_capi.TD_TIME_PHASES)
        barrier(world)
        phases = [round(max_over_ranks(x, world) * 1000.0, 2) for x in w.phase_times()]

    # ---- N > 1: the paper-literal NCCL combine and the ring pass-KV schedule on the
    # same cache, fewer steps (the reference's run_sweep times tree and ring for
    # every cell, bench.cpp:83-112)
    compare = None
    if world > 1 and args.algo == "tree" and not args.no_compare:
        def timed_loop(fn, steps):
            for _ in range(2):
                fn(0)
            barrier(world)
            align_streams(world, stream)
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            ea.record(stream)
            for i in range(steps):
                if flush:
                    fe[i][0].record(stream)
                    with torch.cuda.stream(stream):
                        flush_l2()
                    fe[i][1].record(stream)
                fn(0)
            eb.record(stream)
            barrier(world)
            f_ms = sum(x.elapsed_time(y) for x, y in fe) if flush else 0.0
            return max_over_ranks((ea.elapsed_time(eb) - f_ms) / steps, world)

        ks = max(3, args.compare_steps)
        nccl_ms = timed_loop(lambda fl: w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), args.scale, fl), ks)
        w.reset_kernel_timer()
        align_streams(world, stream)
        for _ in range(ks):
            w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), args.scale, _capi.TD_TIME_PHASES)
        barrier(world)
        nccl_phases = [round(max_over_ranks(x, world) * 1000.0, 2) for x in w.phase_times()]
        graph_ms = timed_loop(lambda fl: w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), args.scale,
                                                             fl | _capi.TD_GRAPH), ks)
        try:
            ndev_ms = timed_loop(lambda fl: w.tree_decode_async(q.data_ptr(), n_q, out.data_ptr(), args.scale,
                                                                fl | _capi.TD_NCCL_DEVICE), ks)
        except td.TreeDecError as e:  # no NCCL device API on this box: every rank fails alike
            ndev_ms, ndev_err = None, str(e)
        else:
            ndev_err = None
        ring_ms = timed_loop(lambda fl: w.ring_decode_async(q.data_ptr(), n_q, out.data_ptr(), args.scale, fl), ks)
        compare = {
            "steps": ks,
            "tree_us": ms * 1000.0, "tree_combine": args.combine,
            "nccl_us": nccl_ms * 1000.0,
            "nccl_phases_us": dict(zip(("K1", "K2", "allreduce_max", "K3", "allreduce_sum", "K4"), nccl_phases)),
            "nccl_graph_us": graph_ms * 1000.0,
            "nccl_device_us": ndev_ms * 1000.0 if ndev_ms is not None else None,
            **({"nccl_device_error": ndev_err} if ndev_err else {}),
            "ring_us": ring_ms * 1000.0,
            "tree_over_ring": ring_ms / ms,
            "note": "same cache and query; nccl = K1, K2, ncclAllReduce(max), K3, ncclAllReduce(sum), K4 "
                    "(decode.cpp:129-173 literally), nccl_graph = the same step replayed as a CUDA graph; "
                    "nccl_device = the same two allreduces inside one combine kernel through NCCL's device API "
                    "(symmetric window, ncclGetLsaPointer); ring = p-1 NCCL send/recv rotations of the KV shards with "
                    "the partial of the chunk in hand overlapped (decode.cpp:186-251); tree_over_ring = "
                    "ring_us / tree_us",
        }

    # ---- parity of the timed output (rank 0; the checker, not the product)
    parity = None
    if rank == 0 and not args.no_parity:
        try:
            parity = parity_leg(args, wl, q, out_timed, world)
        except Exception as e:  # the oracle library may be absent on a foreign box
            parity = {"max_rel_err": None, "ok": False, "note": f"unavailable: {e}"}
    barrier(world)

    # ---- CPU reference baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            heads = args.cpu_sample_heads or min(b * n_q, os.cpu_count() or 1)
            vals, info = reference_cpu(args, wl, 1, heads, os.cpu_count() or 1, steps=3)
            cpu = {"value": min(vals), "unit": "µs/token", "cores": info["cores"], "kind": "reference",
                   "sample": info["sample"] + f"; host nproc={os.cpu_count()}, {cpu_model()}"}
            # the same reference, one row on one thread (threads=p and 1)
            vals1, info1 = reference_cpu(args, wl, 1, 1, 1, steps=2)
            cpu["one_thread"] = {"value": min(vals1), "cores": 1, "sample": info1["sample"]}
        except Exception as e:  # the reference library may be absent on a foreign box
            cpu = {"value": None, "unit": "µs/token", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        peak, peak_kind = load_peaks()
        kv_per_rank = 2 * b * n_kv * math.ceil(n / world) * d * esz
        achieved = kv_per_rank / (k1_ms_max * 1e-3) / 1e9 if k1_ms_max > 0 else None
        # latency per decoded token = the step: each of the b sequences gets its
        # next token when the step ends (b = 1 at the default workload)
        line = {
            "metric": METRIC, "value": ms * 1000.0, "unit": "µs/token", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": dt,
            "data": "synthetic (reference SplitMix64 generator, generated on device)",
            "config": bench_config(args, wl, world,
                                   args.combine if world > 1 and args.algo == "tree" else "none", flush),
            "hbm_gbs_step": kv_per_rank / (ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None,
                         "traffic": load_traffic(args.workload, args.algo, math.ceil(n / world)),
                         "kernel": {1: "k1_bf16 (split-KV, TMA + mma.sync)", 2: "k1_f32 (split-KV, bulk copy)",
                                    0: "k1_generic"}.get(split_kernel), "kernel_ms": k1_ms_max,
                         "bytes_per_launch": kv_per_rank, "peak_kind": peak_kind,
                         "step_frac": kv_per_rank / (ms * 1e-3) / 1e9 / peak,
                         "read_ceiling": read_ceiling(kv_per_rank)},
            "cpu_baseline": cpu,
            "parity": parity,
            "compare": compare,
            "ring_us": compare["ring_us"] if compare else None,
            "nccl_us": compare["nccl_us"] if compare else None,
            "nccl_device_us": compare["nccl_device_us"] if compare else None,
            "tree_over_ring": compare["tree_over_ring"] if compare else None,
            "sequences_per_s": b / (ms * 1e-3),
            "e2e": {"value": e2e_ms * 1000.0, "unit": "µs/token",
                    "h2d_bytes_per_step": q.numel() * esz, "d2h_bytes_per_step": out.numel() * 4,
                    "matches_device_output": bool(ok)},
            "interconnect": interconnect(args, world, b, n_q, n_kv, n, d, esz, ms),
            "memory": {"library_bytes_max_rank": int(lib_bytes), "device_used_bytes_max_rank": int(used_max),
                       "kv_bytes_per_rank": kv_per_rank},
            "calibration": dict(zip(("gain", "state"), w.calibration_info())),
            "phases_us": phases,
            "gpu_launches": kernels_per_step * args.steps,
            "kernels_per_step": kernels_per_step,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if base_flags and w.p2p_status():
        print("p2p exchange reported a timeout", file=sys.stderr)
        sys.exit(3)
    w.close()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

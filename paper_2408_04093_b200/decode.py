"""Host-side mirror of the reference decode API (namespace treedec,
/root/reference/proj/core/include/treedec/decode.hpp) over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference:

* ``chunk_extents`` / ``shard_kv``       attention.cpp:268-275, decode.cpp:68-85
* ``attention_chunk_partial``            attention.cpp:146-168
* ``combine_partials`` / ``combine_pair`` / ``partial_to_numerator``
                                          attention.cpp:178-266
* ``tree_decode`` / ``ring_decode``      decode.cpp:100-251 (single process,
  p workers on one GPU, like the reference's in-process workers)
* ``Worker``                             one rank of the real multi-GPU path
  (one process per GPU, NCCL over NVLink)
* cost counters                          cluster.cpp:106-131 closed forms

Shape errors raise ``InvalidArgument`` (a ``ValueError``), like the
reference's ``std::invalid_argument``. Every computation runs in
libtreedec_b200.so; torch only provides device memory and streams.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

from . import _capi
from ._capi import InvalidArgument, check, lib


class DType(enum.IntEnum):  # dtype.hpp:13
    Float64 = 0
    Float32 = 1
    Bf16 = 2


class ReduceStrategy(enum.IntEnum):  # reduce.hpp:10
    TreeBinary = 0
    Ring = 1
    Hierarchical = 2


class DecodeAlgo(enum.IntEnum):  # cluster.hpp:241
    Ring = 0
    Tree = 1


def _torch():
    import torch
    return torch


def torch_dtype(dt: DType):
    torch = _torch()
    return {DType.Float64: torch.float64, DType.Float32: torch.float32, DType.Bf16: torch.bfloat16}[DType(dt)]


def dtype_of(t) -> DType:
    torch = _torch()
    m = {torch.float64: DType.Float64, torch.float32: DType.Float32, torch.bfloat16: DType.Bf16}
    if t.dtype not in m:
        raise InvalidArgument(_capi.TD_EINVAL, f"unsupported dtype {t.dtype}")
    return m[t.dtype]


def set_deterministic(on: bool = True) -> None:
    """On (the default): the static, calibrated split -- bitwise-reproducible
    results like the reference's (test_decode.cpp:185-202). Off: every call
    hands the last ~15% of each (batch, kv-head) row out dynamically to the SMs
    that stream fastest (TD_DYNAMIC); results then agree to ~1e-7 between calls."""
    check(lib().td_set_deterministic(1 if on else 0))


def _stream_ptr():
    return _torch().cuda.current_stream().cuda_stream


# ---------------------------------------------------------------- host logic
def chunk_extents(n: int, p: int) -> list[int]:
    """ceil(n/p) for the first n % p chunks, floor(n/p) for the rest."""
    if p < 1:
        raise InvalidArgument(_capi.TD_EINVAL, "chunk_extents: p must be >= 1")
    if n < 0:
        raise InvalidArgument(_capi.TD_EINVAL, "chunk_extents: negative length")
    base, rem = divmod(n, p)
    return [base + (1 if i < rem else 0) for i in range(p)]


def shard_range(n: int, p: int, w: int) -> tuple[int, int]:
    """[start, start+len) of worker w's contiguous chunk (decode.cpp:68-85)."""
    ext = chunk_extents(n, p)
    return sum(ext[:w]), ext[w]


@dataclass
class Topology:  # cluster.hpp:172-183 (link parameters are not modelled on the GPU path)
    nodes: int = 1
    gpus_per_node: int = 8

    def world_size(self) -> int:
        return self.nodes * self.gpus_per_node


def topology_for_workers(workers: int) -> Topology:  # cluster.cpp:11-22
    if workers < 1:
        raise InvalidArgument(_capi.TD_EINVAL, "topology_for_workers: workers must be >= 1")
    if workers <= 8:
        return Topology(1, workers)
    if workers % 8:
        raise InvalidArgument(_capi.TD_EINVAL, "topology_for_workers: workers not a multiple of gpus_per_node")
    return Topology(workers // 8, 8)


def peak_memory_formula(algo: DecodeAlgo, b: int, t: int, d: int, n_h: int) -> int:  # cluster.cpp:106-114
    if algo == DecodeAlgo.Ring:
        return 4 * b * t * d + 2 * b * d
    return 2 * b * t * d + 2 * b * d + 2 * b * n_h


def comm_volume_formula(algo: DecodeAlgo, b: int, t: float, d: int, n_h: int, p: int) -> float:  # :116-124
    if algo == DecodeAlgo.Ring:
        return 2.0 * b * t * d * p
    return 2.0 * (p - 1) / p * (b * d + 2.0 * b * n_h)


def comm_volume_formula_seq(algo: DecodeAlgo, b: int, seq_len: int, d: int, n_h: int, p: int) -> float:
    if algo == DecodeAlgo.Ring:
        return float(2 * b * d * seq_len)
    return comm_volume_formula(algo, b, 0.0, d, n_h, p)


def _ceil_log2(p: int) -> int:  # reduce.cpp:24-27
    return 0 if p <= 1 else (p - 1).bit_length()


def allreduce_rounds(strategy: ReduceStrategy, nodes: int, gpus_per_node: int) -> tuple[int, int]:
    """(reduce rounds, total rounds) of allreduce_schedule (reduce.cpp:60-139):
    TreeBinary ceil(log2 p) + its broadcast, Ring (p-1) + (p-1), Hierarchical
    (g-1) intra + ceil(log2 nodes) inter, mirrored. Every strategy moves
    2(p-1) transfers in total; only the round count differs."""
    if nodes < 1 or gpus_per_node < 1:
        raise InvalidArgument(_capi.TD_EINVAL, "allreduce_schedule: bad topology")
    p = nodes * gpus_per_node
    strategy = ReduceStrategy(strategy)
    if strategy == ReduceStrategy.TreeBinary:
        r = _ceil_log2(p)
        return r, 2 * r
    if strategy == ReduceStrategy.Ring:
        return p - 1, 2 * (p - 1)
    r = (gpus_per_node - 1) + _ceil_log2(nodes)
    return r, 2 * r


def ring_schedule(p: int) -> list[list[tuple[int, int, int]]]:
    """Per round r: (worker, chunk held, chunk received) -- decode.cpp:213-238."""
    return [[(w, (w - r) % p, (w - 1 - r) % p) for w in range(p)] for r in range(p - 1)]


def ring_fold_order(p: int, w: int = 0) -> list[int]:
    """Chunk order worker w folds: its own chunk, then w-1, w-2, ... (decode.cpp:214-237)."""
    return [(w - r) % p for r in range(p)]


@dataclass
class CostAccount:  # cluster.hpp:197-212, reporting conventions of decode.cpp:48-62
    elems_sent_intra: float = 0.0
    elems_sent_inter: float = 0.0
    wire_elems_intra: int = 0
    wire_elems_inter: int = 0
    rounds: int = 0
    peak_elems_per_worker: int = 0

    def elems_sent_total(self) -> float:
        return self.elems_sent_intra + self.elems_sent_inter

    def wire_elems_total(self) -> int:
        return self.wire_elems_intra + self.wire_elems_inter


def tree_cost(b: int, n_q: int, n_kv: int, seq_len: int, d_h: int, p: int,
              strategy: ReduceStrategy = ReduceStrategy.Hierarchical, topo: Topology | None = None) -> CostAccount:
    """Counters of one tree decode step (decode.cpp:110-177): convention volume
    2(p-1)/p (b d + 2 b n_h); wire = 2(p-1) (b d + 2 b n_h) (every allreduce
    schedule moves 2(p-1) transfers of each payload); rounds = two collectives
    of the strategy's schedule; peak = Mem_tree with GQA-corrected KV (n_kv heads)."""
    d = n_q * d_h
    t = math.ceil(seq_len / p)
    topo = topo or topology_for_workers(p)
    vol = comm_volume_formula_seq(DecodeAlgo.Tree, b, seq_len, d, n_q, p)
    wire = 2 * (p - 1) * (b * d + 2 * b * n_q)
    rounds = 2 * allreduce_rounds(strategy, topo.nodes, topo.gpus_per_node)[1]
    peak = 2 * b * t * n_kv * d_h + 2 * b * d + 2 * b * n_q
    return CostAccount(vol, 0.0, wire, 0, rounds, peak)


def tree_collectives(strategy: ReduceStrategy, topo: Topology) -> list[tuple[int, int]]:
    """DecodeResult.collectives of tree_decode (decode.cpp:140-142, 161-162):
    (reduce rounds, broadcast rounds) of the max and of the fused sum allreduce."""
    red, tot = allreduce_rounds(strategy, topo.nodes, topo.gpus_per_node)
    return [(red, tot - red)] * 2


def ring_cost(b: int, n_q: int, n_kv: int, seq_len: int, d_h: int, p: int) -> CostAccount:
    d_kv = n_kv * d_h
    t = math.ceil(seq_len / p)
    vol = float(2 * b * d_kv * seq_len) if p > 1 else 0.0
    wire = 2 * b * d_kv * seq_len * (p - 1)
    peak = 4 * b * t * d_kv + 2 * b * n_q * d_h if p > 1 else 2 * b * t * d_kv + 2 * b * n_q * d_h
    return CostAccount(vol, 0.0, wire, 0, p - 1, peak)


# ---------------------------------------------------------------- device primitives
def seeded_tensor(shape, seed: int, scale: float = 1.0, dtype: DType = DType.Bf16, device="cuda",
                  start: int = 0, length: int | None = None):
    """seeded_random_tensor(shape, seed, scale, dtype) on the device, bit-exact
    (numerics.cpp:41-50). shape is [..., seq, d]; with start/length only rows
    [start, start+length) of the seq axis are produced (a shard)."""
    torch = _torch()
    shape = list(shape)
    if len(shape) < 2:
        shape = [1] * (2 - len(shape)) + shape
    *lead, seq, d = shape
    bh = math.prod(lead) if lead else 1
    length = seq - start if length is None else length
    out = torch.empty(*lead, length, d, dtype=torch_dtype(dtype), device=device)
    check(lib().td_seeded_fill(int(dtype), out.data_ptr(), seed, scale, bh, seq, start, length, d, _stream_ptr()))
    return out


@dataclass
class SoftmaxPartial:  # attention.hpp:22-30 (fp32 on the device)
    row_max: object
    lse: object
    out: object


def _check_qkv(q, k, v, what):
    if q.dim() != 3 or k.dim() != 4 or v.shape != k.shape:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: q [b,n_q,d] and k/v [b,n_kv,t,d] required")
    if k.shape[0] != q.shape[0] or k.shape[3] != q.shape[2] or q.shape[1] % k.shape[1]:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: q/k shape mismatch")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: dtype mismatch")
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: tensors must live on the GPU")


def attention_chunk_partial(q, k, v, scale: float = 1.0) -> SoftmaxPartial:
    """q [b, n_q, d], k/v [b, n_kv, t, d] (contiguous, bf16 or f32) -> fp32 partial."""
    torch = _torch()
    _check_qkv(q, k, v, "attention_chunk_partial")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    b, n_q, d = q.shape
    n_kv, t = k.shape[1], k.shape[2]
    ws = _ctypes_size()
    check(lib().td_decode_workspace_bytes(int(dtype_of(q)), b, n_q, n_kv, t, d, ws))
    work = torch.empty(max(ws.value, 16), dtype=torch.uint8, device=q.device)
    rm = torch.empty(b, n_q, dtype=torch.float32, device=q.device)
    lse = torch.empty(b, n_q, dtype=torch.float32, device=q.device)
    out = torch.empty(b, n_q, d, dtype=torch.float32, device=q.device)
    check(lib().td_decode_partial(int(dtype_of(q)), q.data_ptr(), k.data_ptr(), v.data_ptr(), b, n_q, n_kv, t, d,
                                  float(scale), rm.data_ptr(), lse.data_ptr(), out.data_ptr(), work.data_ptr(),
                                  work.numel(), _stream_ptr()))
    return SoftmaxPartial(rm, lse, out)


# ---------------------------------------------------------------- energy formulation
@dataclass
class EnergyEval:  # energy.hpp:16-18: per query row, fp32 on the device, natural log
    value: object        # logsumexp_a(q.k_a + source.v_a) = shifted_lse + row_max
    row_max: object
    shifted_lse: object


def _check_energy(q, k, v, source, what):
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: rank-4 tensors required")
    if k.shape[0] != q.shape[0] or k.shape[1] != q.shape[1] or k.shape[3] != q.shape[3]:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: q/k shape mismatch")
    if v.shape != k.shape:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: k/v shape mismatch")
    if source is not None and source.shape != q.shape:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: source must have the query shape")
    if dtype_of(q) != dtype_of(k) or dtype_of(k) != dtype_of(v) or (source is not None and dtype_of(source) != dtype_of(q)):
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: mixed dtypes")


def energy_partial(q, k, v, source=None) -> SoftmaxPartial:
    """One key chunk of the energy (energy.cpp:27-47 scores q.k_a + source.v_a,
    no 1/sqrt(d) scale): per row (row_max, lse, out), q/source [b, h, nq, d],
    k/v [b, h, t, d]."""
    torch = _torch()
    _check_energy(q, k, v, source, "energy_partial")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    src = None if source is None else source.contiguous()
    b, h, nq, d = q.shape
    t = k.shape[2]
    ws = _ctypes_size()
    check(lib().td_energy_workspace_bytes(int(dtype_of(q)), b, h, nq, t, d, ws))
    work = torch.empty(max(ws.value, 16), dtype=torch.uint8, device=q.device)
    rm = torch.empty(b, h, nq, dtype=torch.float32, device=q.device)
    lse = torch.empty(b, h, nq, dtype=torch.float32, device=q.device)
    out = torch.empty(b, h, nq, d, dtype=torch.float32, device=q.device)
    check(lib().td_energy_partial(int(dtype_of(q)), q.data_ptr(), None if src is None else src.data_ptr(),
                                  k.data_ptr(), v.data_ptr(), b, h, nq, t, d, rm.data_ptr(), lse.data_ptr(),
                                  out.data_ptr(), work.data_ptr(), work.numel(), _stream_ptr()))
    return SoftmaxPartial(rm, lse, out)


def _energy_chunks(k, v, chunks, what):
    n = k.shape[2]
    if chunks < 1 or chunks > n:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: need 1 <= chunks <= N")
    begin = 0
    for ext in chunk_extents(n, chunks):
        yield k[:, :, begin:begin + ext], v[:, :, begin:begin + ext]
        begin += ext


def energy_forward_parallel(q, k, v, source=None, chunks: int = 1) -> EnergyEval:
    """energy_forward_parallel (energy.cpp:152-203): the key axis in `chunks`
    pieces, local (max, lse) per piece, then the max and logsumexp reductions.
    Equal to the one-chunk energy for every chunk count."""
    torch = _torch()
    _check_energy(q, k, v, source, "energy_forward_parallel")
    parts = [energy_partial(q, kc, vc, source) for kc, vc in _energy_chunks(k, v, chunks, "energy_forward_parallel")]
    rows = parts[0].lse.numel()
    rm = torch.stack([p.row_max.reshape(-1) for p in parts]).contiguous()
    lse = torch.stack([p.lse.reshape(-1) for p in parts]).contiguous()
    shape = parts[0].lse.shape
    value, row_max, shifted = (torch.empty(shape, dtype=torch.float32, device=q.device) for _ in range(3))
    check(lib().td_energy_combine(len(parts), rm.data_ptr(), lse.data_ptr(), rows, value.data_ptr(),
                                  row_max.data_ptr(), shifted.data_ptr(), _stream_ptr()))
    return EnergyEval(value, row_max, shifted)


def energy(q, k, v, source=None) -> EnergyEval:
    """energy (energy.cpp:63-83): the one-chunk forward."""
    return energy_forward_parallel(q, k, v, source, 1)


def energy_grad_parallel(q, k, v, saved: EnergyEval, chunks: int = 1):
    """energy_grad_parallel (energy.cpp:205-259): the source-free gradient
    replaying `saved`, sum_a e^(q.k_a - row_max - shifted) v_a per chunk, summed
    over chunks. Equals the attention output."""
    torch = _torch()
    _check_energy(q, k, v, None, "energy_grad_parallel")
    b, h, nq, d = q.shape
    if tuple(saved.row_max.shape) != (b, h, nq) or tuple(saved.shifted_lse.shape) != (b, h, nq):
        raise InvalidArgument(_capi.TD_EINVAL, "energy_grad_parallel: saved evaluation does not match inputs")
    parts = [energy_partial(q, kc, vc, None) for kc, vc in _energy_chunks(k, v, chunks, "energy_grad_parallel")]
    rows = b * h * nq
    lse = torch.stack([p.lse.reshape(-1) for p in parts]).contiguous()
    out = torch.stack([p.out.reshape(rows, d) for p in parts]).contiguous()
    grad = torch.empty(b, h, nq, d, dtype=torch.float32, device=q.device)
    rm = saved.row_max.to(torch.float32).contiguous()
    sh = saved.shifted_lse.to(torch.float32).contiguous()
    check(lib().td_energy_grad_combine(len(parts), lse.data_ptr(), out.data_ptr(), rm.data_ptr(), sh.data_ptr(),
                                       rows, d, grad.data_ptr(), _stream_ptr()))
    return grad


def _ctypes_size():
    import ctypes
    return ctypes.c_size_t()


def combine_partials(parts: list[SoftmaxPartial]):
    """Exact n-way combine (attention.cpp:207-241); InvalidArgument if a row
    attends no key."""
    torch = _torch()
    if not parts:
        raise InvalidArgument(_capi.TD_EINVAL, "combine_partials: no parts")
    first = parts[0].out
    for p in parts:
        if p.out.shape != first.shape:
            raise InvalidArgument(_capi.TD_EINVAL, "combine_partials: shape mismatch")
    d = first.shape[-1]
    rows = first.numel() // d
    lse = torch.stack([p.lse.reshape(-1) for p in parts]).contiguous()
    out = torch.stack([p.out.reshape(rows, d) for p in parts]).contiguous()
    res = torch.empty_like(first, dtype=torch.float32)
    check(lib().td_combine_partials(len(parts), lse.data_ptr(), out.data_ptr(), rows, d, res.data_ptr(),
                                    _stream_ptr()))
    return res


def partial_to_numerator(part: SoftmaxPartial, shift):
    """(numerator, denominator) against a common shift (attention.cpp:243-266)."""
    torch = _torch()
    if shift.shape != part.lse.shape:
        raise InvalidArgument(_capi.TD_EINVAL, "partial_to_numerator: shift shape mismatch")
    d = part.out.shape[-1]
    rows = part.lse.numel()
    nd = torch.empty(rows * d + rows, dtype=torch.float32, device=part.out.device)
    check(lib().td_partial_to_numerator(part.lse.contiguous().data_ptr(), part.out.contiguous().data_ptr(),
                                        shift.contiguous().data_ptr(), rows, d, nd.data_ptr(), _stream_ptr()))
    return nd[: rows * d].view(part.out.shape), nd[rows * d:].view(part.lse.shape)


def combine_pair(left: SoftmaxPartial, right: SoftmaxPartial) -> SoftmaxPartial:
    """Pairwise merge (attention.cpp:178-205); returns a new partial."""
    if left.out.shape != right.out.shape or left.lse.shape != right.lse.shape:
        raise InvalidArgument(_capi.TD_EINVAL, "combine_pair: shape mismatch")
    res = SoftmaxPartial(left.row_max.clone(), left.lse.clone(), left.out.clone())
    d = left.out.shape[-1]
    check(lib().td_combine_pair(res.row_max.data_ptr(), res.lse.data_ptr(), res.out.data_ptr(),
                                right.row_max.contiguous().data_ptr(), right.lse.contiguous().data_ptr(),
                                right.out.contiguous().data_ptr(), left.lse.numel(), d, _stream_ptr()))
    return res


def finalize(num, den):
    torch = _torch()
    d = num.shape[-1]
    rows = den.numel()
    nd = torch.cat([num.reshape(-1), den.reshape(-1)]).float().contiguous()
    out = torch.empty(num.shape, dtype=torch.float32, device=num.device)
    check(lib().td_finalize(nd.data_ptr(), rows, d, out.data_ptr(), None, _stream_ptr()))
    return out


# ---------------------------------------------------------------- single-process reference API
@dataclass
class ShardedKVCache:  # decode.hpp:15-20
    k_chunks: list
    v_chunks: list
    seq_len: int = 0

    def workers(self) -> int:
        return len(self.k_chunks)


def shard_kv(k, v, p: int) -> ShardedKVCache:
    """Contiguous chunks of the sequence axis (copies, like slice_seq)."""
    if k.dim() != 4 or v.shape != k.shape:
        raise InvalidArgument(_capi.TD_EINVAL, "shard_kv: k/v must be rank-4 with equal shapes")
    n = k.shape[2]
    if p < 1:
        raise InvalidArgument(_capi.TD_EINVAL, "shard_kv: p must be >= 1")
    if p > n:
        raise InvalidArgument(_capi.TD_EINVAL, "shard_kv: more workers than keys")
    cache = ShardedKVCache([], [], n)
    begin = 0
    for ext in chunk_extents(n, p):
        cache.k_chunks.append(k[:, :, begin:begin + ext].contiguous())
        cache.v_chunks.append(v[:, :, begin:begin + ext].contiguous())
        begin += ext
    return cache


@dataclass
class DecodeResult:  # decode.hpp:32-38 (+ fp32 output of the GPU path)
    output: object
    cost: CostAccount = field(default_factory=CostAccount)
    collectives: list = field(default_factory=list)


def _require(q, cache: ShardedKVCache, topo: Topology, what: str):
    if q.dim() != 3 and not (q.dim() == 4 and q.shape[2] == 1):
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: single query row required")
    if cache.workers() == 0:
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: empty cache")
    if cache.workers() != topo.world_size():
        raise InvalidArgument(_capi.TD_EINVAL, f"{what}: cache/topology worker count mismatch")
    return q.reshape(q.shape[0], q.shape[1], q.shape[-1])


def tree_decode(q, cache: ShardedKVCache, topo: Topology, strategy: ReduceStrategy = ReduceStrategy.Hierarchical,
                scale: float = 1.0) -> DecodeResult:
    """Algorithm 3 with p in-process workers on one GPU: per-worker partials
    (K1+K2), then max-shift / rescale / sum / divide fused in one combine
    kernel (the single-device image of the two allreduces)."""
    q3 = _require(q, cache, topo, "tree_decode")
    parts = [attention_chunk_partial(q3, k, v, scale) for k, v in zip(cache.k_chunks, cache.v_chunks)]
    out = combine_partials(parts)
    b, n_q, d = q3.shape
    n_kv = cache.k_chunks[0].shape[1]
    p = cache.workers()
    strategy = ReduceStrategy(strategy)
    return DecodeResult(out, tree_cost(b, n_q, n_kv, cache.seq_len, d, p, strategy, topo),
                        tree_collectives(strategy, topo))


def ring_decode(q, cache: ShardedKVCache, topo: Topology, scale: float = 1.0) -> DecodeResult:
    """Ring pass-KV fold order of the reference (worker 0's root)."""
    q3 = _require(q, cache, topo, "ring_decode")
    p = cache.workers()
    parts = [attention_chunk_partial(q3, k, v, scale) for k, v in zip(cache.k_chunks, cache.v_chunks)]
    root = parts[0]
    for r in range(p - 1):
        root = combine_pair(root, parts[(p - 1 - r) % p])
    b, n_q, d = q3.shape
    n_kv = cache.k_chunks[0].shape[1]
    return DecodeResult(root.out, ring_cost(b, n_q, n_kv, cache.seq_len, d, p), [])


def decode_tolerance_abs(dtype: DType, ref_max_abs: float) -> float:  # decode.cpp:253-260
    if dtype == DType.Float32:
        return 1e-4 * ref_max_abs
    if dtype == DType.Bf16:
        return 2e-2 * ref_max_abs
    return 1e-10


# ---------------------------------------------------------------- p workers in one process
class WorkerGroup:
    """The reference's p in-process workers (decode.hpp:70-72; one thread per
    worker under parallel_workers, decode.cpp:37-41) in ONE process: worker w is
    a Worker on device devices[w * len(devices) // p] (contiguous placement,
    cluster.hpp:18-24), several workers may share a GPU. Place shards through
    ``group.workers[w]`` (generate_kv / place_kv), call ``enable_p2p`` once, then
    ``tree_decode`` runs K1 + the one-shot exchange combine (K2x) on every
    worker, the peers' exchange buffers addressed as plain device pointers."""

    def __init__(self, workers: int, devices=None):
        import ctypes
        torch = _torch()
        if devices is None:
            devices = list(range(max(1, min(workers, torch.cuda.device_count()))))
        arr = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        check(lib().td_group_create(len(devices), arr, workers, ctypes.byref(h)))
        self.h = h
        self.devices = list(devices)
        self.workers = []
        for w in range(workers):
            c = ctypes.c_void_p()
            check(lib().td_group_context(h, w, ctypes.byref(c)))
            self.workers.append(Worker._from_group(c, devices[w * len(devices) // workers]))

    def enable_p2p(self, max_rows: int, d: int):
        check(lib().td_group_p2p_open(self.h, max_rows, d))

    def tree_decode(self, q, scale: float = 1.0, strategy: ReduceStrategy = ReduceStrategy.Hierarchical,
                    out=None, flags: int = 0):
        """Algorithm 3 over the group's workers (decode.cpp:100-184) with the
        one-shot combine; q and out on the host or on worker 0's device."""
        torch = _torch()
        w0 = self.workers[0]
        q = q.reshape(q.shape[0], q.shape[1], q.shape[-1]).contiguous()
        host = not q.is_cuda
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32, device="cpu" if host else q.device, pin_memory=host)
        if host:
            flags |= _capi.TD_HOST_IO
        w0._sync_in(q)
        rc = lib().td_group_tree_decode(self.h, q.data_ptr(), q.shape[1], float(scale), int(strategy),
                                        out.data_ptr(), flags)
        for w in self.workers:
            w._consumed(rc)
        check(rc)
        if not host:
            w0._sync_worker()
            for w in self.workers[1:]:
                w._sync_worker()
            if any(w.p2p_status() for w in self.workers):
                raise _capi.TreeDecError(_capi.TD_ECUDA, "tree_decode: exchange timed out; call enable_p2p again")
        return out

    def tree_decode_async(self, q_ptr: int, n_q: int, out_ptr: int, scale: float = 1.0, flags: int = 0,
                          strategy: int = 2):
        rc = lib().td_group_tree_decode(self.h, q_ptr, n_q, float(scale), strategy, out_ptr, flags)
        for w in self.workers:
            w._consumed(rc)
        check(rc)

    def close(self):
        if getattr(self, "h", None):
            for w in self.workers:
                w.h = None
            lib().td_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- one rank of the multi-GPU path
class Worker:
    """One GPU (one process) holding one contiguous KV shard.

    ``comm`` is None for a world of one, or (nranks, rank, unique_id bytes)
    from ``Worker.unique_id()`` shared by the caller (torch.distributed is the
    plumbing: see ``Worker.from_torch_distributed``)."""

    def __init__(self, device: int = 0, comm: tuple[int, int, bytes] | None = None):
        import ctypes
        self._ct = ctypes
        h = ctypes.c_void_p()
        check(lib().td_create(device, ctypes.byref(h)))
        self.h = h
        self._owned = True  # False: a worker of a WorkerGroup (the group destroys it)
        self.device = device
        self._pending = []  # device tensors an enqueued td_kv_append still reads
        self._live = None   # the last device token: the next decode's split kernel reads it (fused append)
        self._xs = None     # torch handle of the worker's stream (created on first use)
        self._ev = None     # input-ordering event (created on first use)
        self.nranks, self.rank = 1, 0
        if comm is not None:
            nranks, rank, uid = comm
            check(lib().td_comm_init(self.h, nranks, rank, uid))
            self.nranks, self.rank = nranks, rank
        self.n_kv = self.d = self.b = self.seq_len = None
        self.dtype = None

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        buf = ctypes.create_string_buffer(128)
        check(lib().td_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls, device: int):
        import torch.distributed as dist
        nranks, rank = dist.get_world_size(), dist.get_rank()
        if nranks == 1:
            return cls(device)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(device, (nranks, rank, obj[0]))

    def enable_p2p(self, max_rows: int, d: int):
        """Set up the one-shot NVLink exchange (TD_P2P): export this rank's
        exchange-buffer IPC handle, all-gather the handles with
        torch.distributed (plumbing) and map the peers' buffers."""
        import torch.distributed as dist
        h = self._ct.create_string_buffer(64)
        check(lib().td_p2p_handle(self.h, max_rows, d, h))
        handles = [None] * self.nranks
        dist.all_gather_object(handles, h.raw)
        check(lib().td_p2p_open(self.h, b"".join(handles)))

    def p2p_status(self) -> int:
        e = self._ct.c_int()
        check(lib().td_p2p_status(self.h, self._ct.byref(e)))
        return e.value

    @classmethod
    def _from_group(cls, handle, device: int):
        import ctypes
        w = cls.__new__(cls)
        w._ct = ctypes
        w.h = handle
        w._owned = False
        w.device = device
        w._pending, w._xs, w._ev, w._live = [], None, None, None
        n, r = ctypes.c_int(), ctypes.c_int()
        check(lib().td_comm_info(handle, ctypes.byref(n), ctypes.byref(r)))
        w.nranks, w.rank = n.value, r.value
        w.n_kv = w.d = w.b = w.seq_len = None
        w.dtype = None
        return w

    def close(self):
        if getattr(self, "h", None):
            if getattr(self, "_owned", True):
                lib().td_destroy(self.h)  # synchronizes the worker's streams
            self.h = None
        self._pending = []
        self._live = None
        self._xs = None
        self._ev = None

    def _worker_stream(self):
        if self._xs is None:
            self._xs = _torch().cuda.ExternalStream(self.stream, device=self.device)
        return self._xs

    def _sync_worker(self):
        self._worker_stream().synchronize()
        self._pending.clear()

    def _consumed(self, rc: int = 0):
        """A call that reads the cache returned rc: on success a deferred token is now
        read by queued work, so its tensors move to the set held until the next
        synchronisation. After a failure the token may still be deferred: keep it live."""
        if rc == 0 and self._live is not None:
            self._pending.append(self._live)
            self._live = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        s = self._ct.c_void_p()
        check(lib().td_stream(self.h, self._ct.byref(s)))
        return s.value or 0

    def _meta(self, dtype, b, n_kv, seq_len, d):
        self.dtype, self.b, self.n_kv, self.seq_len, self.d = DType(dtype), b, n_kv, seq_len, d

    def generate_kv(self, dtype: DType, b: int, n_kv: int, seq_len: int, d: int, seed_k: int, seed_v: int,
                    scale: float = 1.0):
        """This rank's shard of seeded k/v (bit-exact with the reference generator)."""
        check(lib().td_kv_generate(self.h, int(dtype), b, n_kv, seq_len, d, seed_k, seed_v, scale))
        self._consumed()
        self._meta(dtype, b, n_kv, seq_len, d)

    def place_kv(self, k, v, seq_len: int | None = None, start: int | None = None):
        """Place a [b, n_kv, len, d] shard (torch tensor, host or device) that
        covers rows [start, start+len) of a cache of seq_len tokens."""
        b, n_kv, ln, d = k.shape
        if seq_len is None:
            seq_len = ln * self.nranks
        if start is None:
            start, ext = shard_range(seq_len, self.nranks, self.rank)
            if ext != ln:
                raise InvalidArgument(_capi.TD_EINVAL, "place_kv: shard length does not match chunk_extents")
        k, v = k.contiguous(), v.contiguous()
        if k.is_cuda != v.is_cuda:
            raise InvalidArgument(_capi.TD_EINVAL, "place_kv: k and v must both be on the host or on the device")
        self._sync_in(k)  # the device copy runs on the worker's stream: after k / v's producers
        check(lib().td_kv_place(self.h, int(dtype_of(k)), b, n_kv, seq_len, d, start, ln, k.data_ptr(),
                                v.data_ptr(), 0 if k.is_cuda else 1))
        self._consumed()
        self._meta(dtype_of(k), b, n_kv, seq_len, d)

    def append_kv(self, k, v):
        """Append one token ([b, n_kv, 1, d] or [b, n_kv, d], cache dtype) to the
        cache: every rank calls it, the token lands on rank p-1's shard."""
        if self.rank == self.nranks - 1:
            if dtype_of(k) != self.dtype or dtype_of(v) != self.dtype:
                raise InvalidArgument(_capi.TD_EINVAL, "append_kv: token dtype differs from the cache")
            if k.numel() != self.b * self.n_kv * self.d or v.numel() != k.numel():
                raise InvalidArgument(_capi.TD_EINVAL, "append_kv: token must be [b, n_kv, 1, d]")
            k, v = k.contiguous(), v.contiguous()
            self._sync_in(k)  # k and v come from the same (current) stream
            check(lib().td_kv_append(self.h, k.data_ptr(), v.data_ptr(), 0 if k.is_cuda else 1))
            self._consumed()  # an earlier deferred token is now written by an enqueued kernel
            if k.is_cuda:  # read later on the worker's stream (by the next decode, fused): hold it
                self._live = (k, v)
                if len(self._pending) > 256:
                    self._sync_worker()
        else:
            check(lib().td_kv_append(self.h, None, None, 1))
        self.seq_len += 1

    def energy_forward(self, q, source=None) -> EnergyEval:
        """Alg. 1 over the ranks' shards: q, source [b, n_kv, nq, d] on this
        rank's device -> EnergyEval (identical on every rank)."""
        torch = _torch()
        if q.dim() != 4 or q.shape[0] != self.b or q.shape[1] != self.n_kv or q.shape[3] != self.d:
            raise InvalidArgument(_capi.TD_EINVAL, "energy_forward: q must be [b, kv_heads, nq, d]")
        if source is not None and source.shape != q.shape:
            raise InvalidArgument(_capi.TD_EINVAL, "energy_forward: source must have the query shape")
        q = q.contiguous()
        src = None if source is None else source.contiguous()
        shape = q.shape[:3]
        value, rm, sh = (torch.empty(shape, dtype=torch.float32, device=q.device) for _ in range(3))
        self._sync_in(q)
        rc = lib().td_energy_forward(self.h, q.data_ptr(), None if src is None else src.data_ptr(), q.shape[2],
                                     value.data_ptr(), rm.data_ptr(), sh.data_ptr(), 0)
        self._consumed(rc)
        check(rc)
        self._sync_worker()
        return EnergyEval(value, rm, sh)

    def energy_grad(self, q, saved: EnergyEval):
        """Alg. 2: the source-free gradient from the saved forward (= the
        attention output), identical on every rank."""
        torch = _torch()
        if q.dim() != 4 or q.shape[0] != self.b or q.shape[1] != self.n_kv or q.shape[3] != self.d:
            raise InvalidArgument(_capi.TD_EINVAL, "energy_grad: q must be [b, kv_heads, nq, d]")
        q = q.contiguous()
        rm = saved.row_max.to(torch.float32).contiguous()
        sh = saved.shifted_lse.to(torch.float32).contiguous()
        grad = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        self._sync_in(q)
        rc = lib().td_energy_grad(self.h, q.data_ptr(), q.shape[2], rm.data_ptr(), sh.data_ptr(), grad.data_ptr(), 0)
        self._consumed(rc)
        check(rc)
        self._sync_worker()
        return grad

    def calibration_info(self):
        """(gain, state): K1 time the per-SM calibration saves over the equal split
        and whether its weights are in use (2), kept equal (1), not run (0) or failed (-1)."""
        g, st = self._ct.c_double(), self._ct.c_int()
        check(lib().td_calibration_info(self.h, self._ct.byref(g), self._ct.byref(st)))
        return g.value, st.value

    def reserve_kv(self, tokens: int):
        rc = lib().td_kv_reserve(self.h, int(tokens))
        self._consumed(rc)  # a growth writes a deferred token first
        check(rc)

    def kv_info(self):
        s, n, nb = self._ct.c_int64(), self._ct.c_int64(), self._ct.c_size_t()
        check(lib().td_kv_info(self.h, self._ct.byref(s), self._ct.byref(n), self._ct.byref(nb)))
        return s.value, n.value, nb.value

    def _sync_in(self, x):
        """Order the worker's stream after the work already queued on torch's
        current stream (which produced x): an event wait on the device, no host
        block."""
        if x is not None and x.is_cuda:
            torch = _torch()
            if self._ev is None:  # one event, re-recorded: wait_event captures each recording
                self._ev = torch.cuda.Event()
            self._ev.record(torch.cuda.current_stream(x.device))
            self._worker_stream().wait_event(self._ev)

    def _decode(self, fn, q, scale, out, flags, *extra):
        torch = _torch()
        q = q.reshape(q.shape[0], q.shape[1], q.shape[-1]).contiguous()
        n_q = q.shape[1]
        host = not q.is_cuda
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32, device="cpu" if host else q.device,
                              pin_memory=host)
        elif (out.dtype != torch.float32 or out.is_cuda == host or out.numel() != q.numel()
              or not out.is_contiguous()):
            raise InvalidArgument(_capi.TD_EINVAL, "decode: out must be a contiguous fp32 tensor of q's shape, "
                                                   "on the same side (host / device) as q")
        if host:
            flags |= _capi.TD_HOST_IO
            if out.is_pinned():
                flags |= _capi.TD_PINNED_IO  # the combine kernel writes out in place and signals the host
        self._sync_in(q)
        rc = fn(self.h, q.data_ptr(), n_q, float(scale), *extra, out.data_ptr(), flags)
        self._consumed(rc)
        check(rc)
        if not host:
            self._sync_worker()
            if flags & _capi.TD_P2P and self.p2p_status():
                raise _capi.TreeDecError(_capi.TD_ECUDA, "tree_decode: NVLink exchange timed out (a peer never "
                                                         "delivered its partial); call enable_p2p again on every rank")
        return out

    def tree_decode(self, q, scale: float = 1.0, strategy: ReduceStrategy = ReduceStrategy.Hierarchical,
                    out=None, flags: int = 0):
        """Algorithm 3 across the ranks (decode.cpp:100-184); fp32 output on every rank."""
        L = lib()
        return self._decode(lambda h, qp, nq, sc, st, op, fl: L.td_tree_decode(h, qp, nq, sc, st, op, fl),
                            q, scale, out, flags, int(strategy))

    def ring_decode(self, q, scale: float = 1.0, out=None, flags: int = 0):
        """Ring pass-KV comparison (decode.cpp:186-251)."""
        L = lib()
        return self._decode(lambda h, qp, nq, sc, op, fl: L.td_ring_decode(h, qp, nq, sc, op, fl),
                            q, scale, out, flags)

    # -- async launch (no synchronisation) for timing loops ----------------
    def tree_decode_async(self, q_ptr: int, n_q: int, out_ptr: int, scale: float = 1.0, flags: int = 0,
                          strategy: int = 2):
        rc = lib().td_tree_decode(self.h, q_ptr, n_q, float(scale), strategy, out_ptr, flags)
        self._consumed(rc)
        check(rc)

    def ring_decode_async(self, q_ptr: int, n_q: int, out_ptr: int, scale: float = 1.0, flags: int = 0):
        rc = lib().td_ring_decode(self.h, q_ptr, n_q, float(scale), out_ptr, flags)
        self._consumed(rc)
        check(rc)

    def kernel_time(self) -> tuple[float, int]:
        ms, n = self._ct.c_double(), self._ct.c_int()
        check(lib().td_kernel_time(self.h, self._ct.byref(ms), self._ct.byref(n)))
        return ms.value, n.value

    def phase_times(self) -> list[float]:
        arr = (self._ct.c_double * 8)()
        n, calls = self._ct.c_int(), self._ct.c_int()
        check(lib().td_phase_times(self.h, arr, 8, self._ct.byref(n), self._ct.byref(calls)))
        return [arr[i] for i in range(n.value)]

    def debug_stamps(self, n: int = 8 + 8 * 64) -> list[int]:
        arr = (self._ct.c_uint64 * n)()
        check(lib().td_debug_stamps(self.h, arr, n))
        return list(arr)

    def reset_kernel_timer(self):
        check(lib().td_reset_kernel_timer(self.h))

    def last_launch_stats(self) -> tuple[int, float, int]:
        k, by, sk = self._ct.c_int(), self._ct.c_double(), self._ct.c_int()
        check(lib().td_last_launch_stats(self.h, self._ct.byref(k), self._ct.byref(by), self._ct.byref(sk)))
        return k.value, by.value, sk.value

    def memory_bytes(self) -> int:
        n = self._ct.c_size_t()
        check(lib().td_memory_bytes(self.h, self._ct.byref(n)))
        return n.value

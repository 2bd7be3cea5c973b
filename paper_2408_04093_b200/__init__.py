"""B200-native tree-attention decoding (arXiv 2408.04093).

Drop-in for the reference's decode path (treedec::tree_decode /
ring_decode, /root/reference/proj/core): hand-written sm_100a kernels in
libtreedec_b200.so behind the C-ABI of include/treedec_b200.h; this package
is the host-side mirror of the reference interface over that C-ABI.
"""
from ._capi import DomainError, InvalidArgument, TreeDecError  # noqa: F401
from .decode import (  # noqa: F401
    CostAccount, DecodeAlgo, DecodeResult, allreduce_rounds, tree_collectives, DType, EnergyEval, ReduceStrategy, ShardedKVCache, SoftmaxPartial,
    Topology, energy, energy_forward_parallel, energy_grad_parallel, energy_partial,
    Worker, WorkerGroup, attention_chunk_partial, chunk_extents, combine_pair, combine_partials, comm_volume_formula,
    comm_volume_formula_seq, decode_tolerance_abs, finalize, partial_to_numerator, peak_memory_formula,
    ring_cost, ring_decode, ring_fold_order, ring_schedule, seeded_tensor, set_deterministic, shard_kv, shard_range, tree_cost,
    tree_decode, topology_for_workers,
)

__version__ = "0.1.0"

"""Host-side logic of the product package (no GPU): shard geometry, topology,
ring schedule / fold order and the reporting counters, checked against the
reference's closed forms and (where oracle/_ref exists) its DecodeResult
counters."""
import math

import numpy as np
import pytest

import paper_2408_04093_b200 as td
from conftest import make_inputs
from oracle.oracle import F64, HIER


def test_chunk_extents_and_shard_range(oracle):
    for n in (0, 1, 3, 10, 17, 1 << 20, (1 << 20) + 7):
        for p in (1, 2, 3, 5, 7, 8, 16):
            ext = td.chunk_extents(n, p)
            assert ext == oracle.chunk_extents(n, p)
            assert sum(ext) == n and max(ext) - min(ext) <= 1
            begin = 0
            for w in range(p):
                assert td.shard_range(n, p, w) == (begin, ext[w])
                begin += ext[w]
    with pytest.raises(td.InvalidArgument):
        td.chunk_extents(4, 0)
    with pytest.raises(ValueError):
        td.chunk_extents(-1, 2)


def test_topology_for_workers():
    assert td.topology_for_workers(1).world_size() == 1
    t = td.topology_for_workers(8)
    assert (t.nodes, t.gpus_per_node) == (1, 8)
    t = td.topology_for_workers(32)
    assert (t.nodes, t.gpus_per_node) == (4, 8)
    with pytest.raises(td.InvalidArgument):
        td.topology_for_workers(12)
    with pytest.raises(td.InvalidArgument):
        td.topology_for_workers(0)


def test_ring_schedule_matches_reference_rotation():
    """decode.cpp:213-238: worker w holds (w - r) mod p and receives (w - 1 - r) mod p;
    every chunk visits every worker exactly once."""
    for p in (2, 3, 5, 8):
        sched = td.ring_schedule(p)
        assert len(sched) == p - 1
        seen = {w: {w} for w in range(p)}
        for r, rnd in enumerate(sched):
            for w, held, incoming in rnd:
                assert held == (w - r) % p and incoming == (w - 1 - r) % p
                # what w receives is what w-1 holds
                assert incoming == rnd[(w - 1) % p][1]
                seen[w].add(incoming)
        assert all(s == set(range(p)) for s in seen.values())
        assert td.ring_fold_order(p, 0) == [0] + list(range(p - 1, 0, -1))


def test_closed_forms():
    # cluster.cpp:106-131 at the reference test's numbers (test_decode.cpp:121-183)
    b, n_h, d_h = 1, 2, 4
    d = n_h * d_h
    for p in (2, 4, 8):
        t = 64 // p
        assert td.peak_memory_formula(td.DecodeAlgo.Tree, b, t, d, n_h) == 2 * b * t * d + 2 * b * d + 2 * b * n_h
        assert td.peak_memory_formula(td.DecodeAlgo.Ring, b, t, d, n_h) == 4 * b * t * d + 2 * b * d
        assert td.comm_volume_formula_seq(td.DecodeAlgo.Tree, b, 64, d, n_h, p) == \
            td.comm_volume_formula_seq(td.DecodeAlgo.Tree, b, 1024, d, n_h, p)
        assert td.comm_volume_formula_seq(td.DecodeAlgo.Ring, b, 64, d, n_h, p) == \
            td.comm_volume_formula(td.DecodeAlgo.Ring, b, 64 / p, d, n_h, p)


def test_counters_match_reference(oracle, reference):
    """tree_cost / ring_cost (MHA) equal the reference's DecodeResult counters."""
    b, n_h, d_h, n = 1, 2, 4, 64
    q, k, v = make_inputs(oracle, 7, b, n_h, n_h, n, d_h, F64)
    for p in (1, 2, 4, 8):
        with reference.prepare(q, k, v, p, F64) as pr:
            # counters of a single row call: n_h = 1
            for strategy in (0, 1, 2):
                _, _, ct = pr.decode(0, strategy)
                tc = td.tree_cost(1, 1, 1, n, d_h, p, td.ReduceStrategy(strategy))
                assert ct[0] == pytest.approx(tc.elems_sent_total())
                assert ct[1] == tc.wire_elems_total()
                assert ct[2] == tc.peak_elems_per_worker
                assert ct[3] == tc.rounds
            _, _, cr = pr.decode(1, HIER)
            rc = td.ring_cost(1, 1, 1, n, d_h, p)
            assert cr[0] == pytest.approx(rc.elems_sent_total())
            assert cr[1] == rc.wire_elems_total()
            assert cr[3] == rc.rounds
            if p > 1:
                assert cr[2] == rc.peak_elems_per_worker


def test_tolerance_table():
    assert td.decode_tolerance_abs(td.DType.Float64, 5.0) == 1e-10
    assert td.decode_tolerance_abs(td.DType.Float32, 2.0) == pytest.approx(2e-4)
    assert td.decode_tolerance_abs(td.DType.Bf16, 2.0) == pytest.approx(4e-2)


def test_llama_shape_accounting():
    """Reporting at the north-star shape: per-rank KV bytes and the tree payload."""
    b, n_q, n_kv, n, d = 1, 32, 8, 1 << 20, 128
    p = 8
    kv_bytes = 2 * b * n_kv * math.ceil(n / p) * d * 2
    assert kv_bytes == 536870912  # 537 MB per GPU
    tc = td.tree_cost(b, n_q, n_kv, n, d, p)
    assert tc.elems_sent_total() == pytest.approx(2 * 7 / 8 * (32 * 128 + 2 * 32))
    rc = td.ring_cost(b, n_q, n_kv, n, d, p)
    assert rc.wire_elems_total() == 2 * n_kv * d * n * 7


def test_allreduce_rounds_match_reference_schedules(oracle):
    """allreduce_rounds / tree_collectives equal allreduce_schedule's round counts
    (reduce.cpp:60-139) for every strategy and topology."""
    for strategy in (0, 1, 2):
        for nodes, gpus in ((1, 1), (1, 2), (1, 3), (1, 4), (1, 7), (1, 8), (2, 8), (3, 8), (4, 4)):
            want = oracle.schedule_rounds(strategy, nodes, gpus)
            assert td.allreduce_rounds(td.ReduceStrategy(strategy), nodes, gpus) == want
            red, tot = want
            assert td.tree_collectives(td.ReduceStrategy(strategy), td.Topology(nodes, gpus)) == [(red, tot - red)] * 2

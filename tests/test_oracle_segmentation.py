"""CPU: the oracle's segmentation restatement (partition.hpp:58-307,
pipeline.hpp:131-138) against the SPEC.md partition examples
and hand traces of the reference loop, plus its invariants."""
import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth


def path_graph(n):
    offs = [0]
    cols = []
    for v in range(n):
        nb = [w for w in (v - 1, v + 1) if 0 <= w < n]
        cols += nb
        offs.append(len(cols))
    return np.asarray(offs, np.int32), np.asarray(cols, np.int32)


def test_rng_draws_used_by_the_traces():
    # std::mt19937_64(1)() = 14514284786278117030 (libstdc++; pinned by oracle/rng_ref.cpp)
    assert O.MT19937_64(1)() % 8 == 0
    assert O.MT19937_64(3)() % 5 == 2


def test_partition_path_hand_trace():
    """path 0-1-...-7, k = 2, seed 1 (first seed 0): the farthest vertex is 7;
    cap = int(ceil(8/2) * 1.1) = 4; parts grow alternately from the ends
    (part 0 first on size ties, partition.hpp:122-129) -> [0 0 0 0 1 1 1 1]."""
    offs, cols = path_graph(8)
    p = O.partition_mesh(offs, cols, 2, 1)
    assert p.assignment.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]


def test_partition_k1_single_part():
    """k=1 -> single part containing all vertices."""
    m = synth.small_grid(16, 16, 8, 8, seed=1)
    p = O.partition_mesh(m.adj_offsets, m.adj_cols, 1, 5)
    assert np.all(p.assignment == 0)


def test_partition_invariants_and_errors():
    m = synth.small_grid(20, 20, 10, 10, seed=1)
    for k, seed in ((4, 1), (7, 3), (25, 9)):
        p = O.partition_mesh(m.adj_offsets, m.adj_cols, k, seed)
        sizes = p.part_sizes()
        assert sum(sizes) == m.n and min(sizes) >= 1
        # parts are connected by construction (growth from the seed over edges)
        for part in range(k):
            vs = set(np.nonzero(p.assignment == part)[0].tolist())
            start = next(iter(vs))
            seen, stack = {start}, [start]
            while stack:
                v = stack.pop()
                for w in m.adj_cols[m.adj_offsets[v]:m.adj_offsets[v + 1]]:
                    if w in vs and w not in seen:
                        seen.add(int(w))
                        stack.append(int(w))
            assert seen == vs
    with pytest.raises(O.InvalidArgument, match="part count k must satisfy 1 <= k <= n/4"):
        O.partition_mesh(m.adj_offsets, m.adj_cols, m.n // 4 + 1, 1)


def test_partition_disconnected_component_gets_a_seed():
    """farthest-point seeding picks the unreachable component first
    (partition.hpp:96-104: unreachable = max distance)."""
    o1, c1 = path_graph(8)
    offs = np.concatenate([o1, o1[1:] + o1[-1]]).astype(np.int32)
    cols = np.concatenate([c1, c1 + 8]).astype(np.int32)
    p = O.partition_mesh(offs, cols, 2, 1)  # first seed 14514284786278117030 % 16 = 6
    a, b = set(p.assignment[:8].tolist()), set(p.assignment[8:].tolist())
    assert len(a) == 1 and len(b) == 1 and a != b
    with pytest.raises(O.InvalidArgument, match="partition failed"):
        # three components, k = 2: the third never gets a seed (partition.hpp:116-119)
        o3 = np.concatenate([offs, o1[1:] + offs[-1]]).astype(np.int32)
        c3 = np.concatenate([cols, c1 + 16]).astype(np.int32)
        O.partition_mesh(o3, c3, 2, 1)


def test_expand_overlaps_examples():
    m = synth.small_grid(12, 12, 6, 6, seed=1)
    # k=1, growth=1.0 -> one submesh = whole mesh
    p1 = O.partition_mesh(m.adj_offsets, m.adj_cols, 1, 1)
    mem = O.expand_overlaps(m.adj_offsets, m.adj_cols, p1, 1.0)
    assert len(mem) == 1 and mem[0].tolist() == list(range(m.n))
    p = O.partition_mesh(m.adj_offsets, m.adj_cols, 5, 2)
    mem = O.expand_overlaps(m.adj_offsets, m.adj_cols, p, 1.15)
    nd = int(np.floor(1.15 * max(p.part_sizes())))
    cover = np.zeros(m.n, int)
    for part, ms in enumerate(mem):
        assert ms.size == nd and np.all(np.diff(ms) > 0)
        assert set(np.nonzero(p.assignment == part)[0]).issubset(set(ms.tolist()))  # part retained
        cover[ms] += 1
    assert cover.min() >= 1  # every vertex appears in >= 1 submesh
    with pytest.raises(O.InvalidArgument, match="overlap growth must be >= 1.0"):
        O.expand_overlaps(m.adj_offsets, m.adj_cols, p, 0.9)


def test_expand_overlaps_last_ring_keeps_smallest_ids_and_pads():
    """path 0..9, parts {0..4}, {5..9}: growth 1.5 -> n_d = 7; part 0's rings
    are {5}, {6} -> [0..6]; part 1's rings {4}, {3} -> [3..9].  A part whose
    component is exhausted is padded with the smallest unused ids."""
    offs, cols = path_graph(10)
    p = O.Partition(np.asarray([0] * 5 + [1] * 5, np.int32), 2)
    mem = O.expand_overlaps(offs, cols, p, 1.5)
    assert mem[0].tolist() == list(range(7)) and mem[1].tolist() == list(range(3, 10))
    # two components {0..3} and {4..9}: part 0 = {0..3} grows to 6 by padding with 4, 5
    o1, c1 = path_graph(4)
    o2, c2 = path_graph(6)
    offs2 = np.concatenate([o1, o2[1:] + o1[-1]]).astype(np.int32)
    cols2 = np.concatenate([c1, c2 + 4]).astype(np.int32)
    p2 = O.Partition(np.asarray([0] * 4 + [1] * 6, np.int32), 2)
    mem2 = O.expand_overlaps(offs2, cols2, p2, 1.0)
    assert mem2[0].tolist() == [0, 1, 2, 3, 4, 5] and mem2[1].tolist() == list(range(4, 10))


def test_order_submeshes_examples():
    # single submesh -> [0]
    assert O.order_submeshes([np.arange(4)], 7).tolist() == [0]
    # chain of 5 overlapping submeshes, seed picking id 2 -> [2, 1, 3, 0, 4]
    chain = [np.arange(3 * i, 3 * i + 4) for i in range(5)]
    assert O.order_submeshes(chain, 3).tolist() == [2, 1, 3, 0, 4]
    # two disjoint components -> both appear, the second after the first
    comps = [np.arange(0, 4), np.arange(3, 7), np.arange(10, 14), np.arange(13, 17)]
    seq = O.order_submeshes(comps, 3).tolist()  # initial = 3 % 4... any
    assert sorted(seq) == [0, 1, 2, 3]
    first = {0, 1} if seq[0] in (0, 1) else {2, 3}
    assert set(seq[:2]) == first

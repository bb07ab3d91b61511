"""Pins of the oracle's reverse Cuthill-McKee (oracle.h orc_rcm).

Hand-traced small graphs (the trace is written out next to each case), closed forms
(a relabelled path has bandwidth 1; from a lattice corner the Cuthill-McKee levels
are the anti-diagonals), and BFS-level invariants checked with scipy's BFS.
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse import csgraph

import oracle as O
from paper_2201_05413_b200 import inputs as I


def _graph(n, edges):
    """Symmetric pattern with the diagonal, rows sorted (values: Laplacian, unused)."""
    rows = [[i] for i in range(n)]
    for a, b in edges:
        rows[a].append(b)
        rows[b].append(a)
    rows = [sorted(set(r)) for r in rows]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    col = np.concatenate(rows).astype(np.int64) if n else np.zeros(0, dtype=np.int64)
    return O.Csr(n, rp, col, np.ones(len(col)))


def _bandwidth(A, perm):
    iperm = np.empty(A.n, dtype=np.int64)
    iperm[perm] = np.arange(A.n)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    return int(np.max(np.abs(iperm[rows] - iperm[A.col]))) if A.nnz else 0


def test_rcm_hand_trace_degree_order():
    # deg: 0:3 1:2 2:3 3:2 4:2 5:2 6:2 7:2.  start = 1 (least (deg, id)); BFS(1) levels
    # {1} {0,4} {2,3} {5,6} {7}: ecc 4, x = 7; BFS(7) ecc 4, not larger -> r = 1.
    # CM: 1 -> (4 deg 2, 0 deg 3) -> 4: 2 -> 0: 3 -> 2: 5 -> 3: 6 -> 5: 7.
    # order 1 4 0 2 3 5 6 7, reversed:
    A = _graph(8, [(0, 1), (0, 2), (0, 3), (1, 4), (2, 4), (2, 5), (3, 6), (6, 7), (5, 7)])
    assert O.rcm(A).tolist() == [7, 6, 5, 3, 2, 0, 4, 1]


def test_rcm_hand_trace_peripheral_search_moves():
    # path 1-2-3-4-5 with leaf 0 on 3.  start s = 0 (deg 1); BFS(0): ecc 3, last {1,5} -> x = 1;
    # BFS(1): ecc 4 > 3 -> r = 1, x = 5; BFS(5): ecc 4 -> stop.  CM from 1: 1 2 3 (0 deg 1, 4 deg 2) 5
    A = _graph(6, [(1, 2), (2, 3), (3, 4), (4, 5), (0, 3)])
    assert O.rcm(A).tolist() == [5, 4, 0, 3, 2, 1]


def test_rcm_hand_trace_components_and_isolated():
    # node 5 isolated (deg 0) is the first start; then {0,2,4} from 0 (BFS(0) ecc 2, x = 4,
    # BFS(4) ecc 2 -> r = 0), then {1,3} from 1.  order 5 0 2 4 1 3, reversed:
    A = _graph(6, [(1, 3), (0, 2), (2, 4)])
    assert O.rcm(A).tolist() == [3, 1, 4, 2, 0, 5]


def test_rcm_trivial_sizes():
    assert O.rcm(_graph(0, [])).tolist() == []
    assert O.rcm(_graph(1, [])).tolist() == [0]
    assert O.rcm(_graph(4, [])).tolist() == [3, 2, 1, 0]  # all isolated: id order, reversed


@pytest.mark.parametrize("n,seed", [(50, 1), (1000, 2)])
def test_rcm_relabelled_path_bandwidth_one(n, seed):
    q = I.relabel_order(n, seed)
    iq = np.empty(n, dtype=np.int64)
    iq[q] = np.arange(n)
    A = _graph(n, [(int(iq[i]), int(iq[i + 1])) for i in range(n - 1)])
    p = O.rcm(A)
    assert _bandwidth(A, p) == 1
    # the two endpoints have degree 1; the one with the smaller id starts CM, so it ends RCM
    ends = sorted([int(iq[0]), int(iq[n - 1])])
    assert p[-1] == ends[0] and p[0] == ends[1]


@pytest.mark.parametrize("c", [5, 16, 33])
def test_rcm_lattice_antidiagonals(c):
    # 5-point lattice graph: CM from corner 0 places the anti-diagonals i + j = d in order
    n = c * c
    E = [(j * c + i, j * c + i + 1) for j in range(c) for i in range(c - 1)]
    E += [(j * c + i, (j + 1) * c + i) for j in range(c - 1) for i in range(c)]
    A = _graph(n, E)
    p = O.rcm(A)
    d = (p % c) + (p // c)
    assert np.all(np.diff(d[::-1]) >= 0), "levels must be the anti-diagonals in order"
    assert _bandwidth(A, p) <= c
    assert sorted(p.tolist()) == list(range(n))


def _random_mesh_graph(n, seed):
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    from scipy.spatial import Delaunay
    tri = Delaunay(pts).simplices
    E = set()
    for t in tri:
        for a in range(3):
            u, v = int(t[a]), int(t[(a + 1) % 3])
            E.add((min(u, v), max(u, v)))
    return _graph(n, sorted(E))


@pytest.mark.parametrize("n,seed", [(300, 3), (2000, 4)])
def test_rcm_bfs_level_invariants(n, seed):
    A = _random_mesh_graph(n, seed)
    p = O.rcm(A)
    assert sorted(p.tolist()) == list(range(n))
    G = sp.csr_matrix((np.ones(A.nnz), A.col, A.row_ptr), shape=(n, n))
    cm = p[::-1]
    dist = csgraph.shortest_path(G, unweighted=True, indices=int(cm[0]))
    lv = dist[cm]
    assert np.all(np.diff(lv) >= 0), "Cuthill-McKee order is a BFS order: levels contiguous, increasing"
    # the start is pseudo-peripheral: its eccentricity is at least that of the least-degree node
    deg = np.diff(A.row_ptr) - 1
    s = int(np.lexsort((np.arange(n), deg))[0])
    ecc_s = csgraph.shortest_path(G, unweighted=True, indices=s).max()
    assert lv[-1] >= ecc_s
    # bandwidth of the Delaunay graph drops well below the random numbering's
    assert _bandwidth(A, p) < 0.25 * _bandwidth(A, np.arange(n))


def test_rcm_partition_halos_shrink():
    # N4 multi-GPU: contiguous row blocks of a randomly numbered mesh need almost every
    # remote node as a ghost; of the RCM-ordered mesh, only the block interfaces
    P = O.build_problem("C6", c=12, k=1)
    A = P["A"]
    q = I.relabel_order(A.n, 7)
    Ar = O.Csr(A.n, *I.relabel_csr_numpy(A.row_ptr, A.col, A.val, q))
    p = O.rcm(Ar)
    Ao = O.Csr(A.n, *I.relabel_csr_numpy(Ar.row_ptr, Ar.col, Ar.val, p))
    for G in (2, 4):
        hr = [len(O.halo(Ar, int(b0), int(b1))) for b0, b1 in zip(O.partition(Ar, G)[:-1], O.partition(Ar, G)[1:])]
        ho = [len(O.halo(Ao, int(b0), int(b1))) for b0, b1 in zip(O.partition(Ao, G)[:-1], O.partition(Ao, G)[1:])]
        assert max(ho) < 0.25 * max(hr), (G, ho, hr)

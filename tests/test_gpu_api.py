"""convex_hull_3d on the B200 against the unmodified reference's outputs
(tests/golden/small.npz) and its API contract (pkg/tests/test_api.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1205_1171_b200 as H
from paper_1205_1171_b200.generators import generate

pytestmark = pytest.mark.gpu

TETRA = np.array([[0.0, 0, 0], [1, 0.1, 2], [2, 1.9, 0.3], [3, 0.2, 0.1]])


@pytest.mark.parametrize("engine", ["fast", "exact"])
def test_golden_cases_bit_exact(small, engine):
    be = H.CudaBackend(0, engine=engine)
    for name in small.names:
        c = small.case(name)
        if engine == "fast" and not c["general"]:
            continue  # degenerate inputs: the reference's own solvers disagree
        r = H.convex_hull_3d(c["pts"], be)
        assert np.array_equal(r.faces, c["faces"]), name
        assert np.array_equal(r.vertices, c["vertices"]), name
        assert (r.stats.lower_events, r.stats.upper_events) == (c["lower"], c["upper"]), name
        assert r.stats.perturbed == c["perturbed"], name


def test_degenerate_golden_cases_exact_engine(small):
    be = H.CudaBackend(0, engine="exact")
    for name in small.names:
        c = small.case(name)
        if c["general"]:
            continue
        r = H.convex_hull_3d(c["pts"], be)
        assert np.array_equal(r.faces, c["faces"]), name


def test_tetrahedron_and_orientation():
    res = H.convex_hull_3d(TETRA)
    assert res.vertices.tolist() == [0, 1, 2, 3]
    assert len(res.faces) == 4
    c = TETRA.mean(axis=0)
    a = TETRA[res.faces[:, 0]]
    nrm = np.cross(TETRA[res.faces[:, 1]] - a, TETRA[res.faces[:, 2]] - a)
    assert (np.einsum("ij,ij->i", nrm, c - a) < 0).all()


def test_input_order_invariance():
    pts = generate(48, "gauss", 17)
    res = H.convex_hull_3d(pts)
    perm = np.random.default_rng(0).permutation(len(pts))
    res2 = H.convex_hull_3d(pts[perm])
    remapped = {tuple(sorted(int(perm[i]) for i in f)) for f in res2.faces}
    assert remapped == res.face_set()


def test_device_resident_and_pinned_inputs():
    pts = generate(5000, "ball", 1)
    ref = H.convex_hull_3d(pts)
    d = H.convex_hull_3d(torch.from_numpy(pts).cuda(), return_device=True)
    assert d.faces.is_cuda and np.array_equal(d.faces.cpu().numpy(), ref.faces)
    p = H.convex_hull_3d(torch.from_numpy(pts).pin_memory())
    assert np.array_equal(p.faces, ref.faces)


def test_degenerate_inputs_raise():
    rng = np.random.default_rng(1)
    flat = np.column_stack([rng.random(10), rng.random(10), np.zeros(10)])
    with pytest.raises(H.DegenerateInputError):
        H.convex_hull_3d(flat)
    line = np.column_stack([np.arange(8.0), np.arange(8.0) * 2, np.arange(8.0) * 3])
    with pytest.raises(H.DegenerateInputError):
        H.convex_hull_3d(line)
    with pytest.raises(H.DegenerateInputError):
        H.convex_hull_3d(np.zeros((6, 3)))


def test_input_validation():
    with pytest.raises(ValueError, match="no points"):
        H.convex_hull_3d(np.empty((0, 3)))
    with pytest.raises(ValueError):
        H.convex_hull_3d(np.array([[0.0, 0.0]]))
    with pytest.raises(ValueError):
        H.convex_hull_3d(np.array([[0.0, np.inf, 0.0]]))
    with pytest.raises(ValueError, match="finite"):
        H.convex_hull_3d(np.vstack([TETRA, [[np.nan, 0, 0]]]))
    with pytest.raises(ValueError):
        H.convex_hull_3d(TETRA, solver="fancy")


def test_tiny_inputs_have_no_faces():
    for n in (1, 2, 3):
        res = H.convex_hull_3d(generate(n, "gauss", 0))
        assert res.vertices.tolist() == list(range(n))
        assert res.faces.shape == (0, 3)
        assert res.stats.levels == 0


def test_stats_fields():
    pts = generate(256, "ball", 0)
    st = H.convex_hull_3d(pts).stats
    assert st.n == 256 and st.levels == 8
    assert st.solver == "parallel" and st.workers == 1
    assert st.total_ms > 0 and st.sort_ms >= 0
    assert len(st.lower_level_ms) == st.levels
    assert not st.perturbed
    ser = H.convex_hull_3d(pts, solver="serial").stats
    assert ser.solver == "serial" and ser.lower_level_ms == []


def test_every_point_inside_hull():
    for seed in range(3):
        pts = generate(2000, "gauss", seed)
        res = H.convex_hull_3d(pts)
        scale = float(np.abs(pts).max())
        a = pts[res.faces[:, 0]]
        nrm = np.cross(pts[res.faces[:, 1]] - a, pts[res.faces[:, 2]] - a)
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        dist = nrm @ pts.T - np.einsum("ij,ij->i", nrm, a)[:, None]
        assert dist.max() <= 1e-9 * scale
        assert len(res.faces) == 2 * len(res.vertices) - 4


def test_concurrent_threads_one_device(oracle_mod):
    """Hulls from several Python threads on one device (shared workspaces)
    are serialised per device and all correct."""
    import threading

    import numpy as np

    import paper_1205_1171_b200 as H
    from paper_1205_1171_b200.generators import generate

    clouds = [generate(30000 + 17 * i, ("ball", "sphere", "cube")[i % 3], i) for i in range(6)]
    exp = [oracle_mod.convex_hull_3d(p).faces for p in clouds]
    got = [None] * len(clouds)

    def run(i):
        got[i] = H.convex_hull_3d(clouds[i]).faces

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(clouds))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for g, e in zip(got, exp):
        assert np.array_equal(g, e)


def test_stream_api_equals_per_call(oracle_mod):
    """convex_hull_3d_stream (copy of cloud i+1 overlapping hull i) yields,
    in order, exactly what one convex_hull_3d call per cloud returns --
    pinned tensors, numpy arrays and clouds of different sizes mixed."""
    clouds = [torch.from_numpy(generate(20000, "ball", 1)).pin_memory(),
              generate(7777, "cube", 2),
              torch.from_numpy(generate(20000, "sphere", 3)).pin_memory(),
              generate(5000, "gauss", 4)]
    got = list(H.convex_hull_3d_stream(clouds))
    assert len(got) == len(clouds)
    for c, r in zip(clouds, got):
        pts = c.numpy() if isinstance(c, torch.Tensor) else c
        exp = oracle_mod.convex_hull_3d(pts)
        assert np.array_equal(r.faces, exp.faces)
        assert np.array_equal(r.vertices, exp.vertices)
    assert list(H.convex_hull_3d_stream([])) == []


def test_stats_level_times_from_device_stamps():
    """Per-level seconds (HullStats.*_level_ms, F12) come from the level
    kernels' device time stamps: one entry per level, non-negative, and the
    fused leaf levels report at their last level."""
    pts = generate(1 << 16, "ball", 7)
    r = H.convex_hull_3d(pts)
    L = r.stats.levels
    assert len(r.stats.lower_level_ms) == L and len(r.stats.upper_level_ms) == L
    assert all(t >= 0.0 for t in r.stats.lower_level_ms)
    assert sum(r.stats.lower_level_ms) > 0.0
    assert r.stats.lower_level_ms[0] == 0.0 and r.stats.lower_level_ms[2] > 0.0  # leaf: levels 1..3
    assert r.stats.sort_ms > 0.0 and r.stats.lower_ms > 0.0


@pytest.mark.parametrize("case", ["short_runs", "long_run", "perturbed_descends"])
def test_tie_path_variants(case, oracle_mod):
    """The device tie path (api.py:86-110): lexsort by re-ordering the runs
    of equal x (short runs), the three full stable passes (a run longer than
    64), and the stable re-sort after the perturbation when a perturbed x
    overtakes the next distinct x (otherwise the re-sort is the identity)."""
    rng = np.random.default_rng(11)
    pts = rng.uniform(-1, 1, (3000, 3))
    if case == "short_runs":
        pts[:600, 0] = np.repeat(rng.uniform(-1, 1, 200), 3)
    elif case == "long_run":
        pts[:100, 0] = 0.25
    else:  # a run at 1.0, the next distinct x two ulps above: base + 16 eps > it
        pts[:5, 0] = 1.0
        pts[5, 0] = np.nextafter(np.nextafter(1.0, 2.0), 2.0)
    rng.shuffle(pts)
    r = H.convex_hull_3d(pts)
    exp = oracle_mod.convex_hull_3d(pts)
    assert r.stats.perturbed and exp.perturbed
    assert np.array_equal(r.faces, exp.faces)
    assert np.array_equal(r.vertices, exp.vertices)


def test_tie_path_repeated_size(oracle_mod):
    """Same-size calls after a call with x ties start on the device tie path
    (hull.cu: presort_ties_async, no host synchronisation); its gate hands
    long runs and a descending perturbed x back to the exact presort and
    raises the degeneracy errors -- every call still equals the oracle,
    including a tie-free cloud on that path (perturbed stays False)."""
    rng = np.random.default_rng(5)

    def cloud(kind):
        pts = rng.uniform(-1, 1, (3000, 3))
        if kind == "short_runs":
            pts[:600, 0] = np.repeat(rng.uniform(-1, 1, 200), 3)
        elif kind == "long_run":
            pts[:100, 0] = 0.25
        elif kind == "perturbed_descends":
            pts[:5, 0] = 1.0
            pts[5, 0] = np.nextafter(np.nextafter(1.0, 2.0), 2.0)
        elif kind == "coplanar_ties":
            pts[:, 2] = 0.0
            pts[:4, 0] = 0.5
        rng.shuffle(pts)
        return pts

    seq = ["short_runs", "short_runs", "none", "short_runs", "long_run", "perturbed_descends",
           "coplanar_ties", "short_runs", "short_runs"]
    for kind in seq:
        pts = cloud(kind)
        try:
            exp = oracle_mod.convex_hull_3d(pts)
        except ValueError as e:  # the oracle's DegenerateInputError: the package's own class
            assert type(e).__name__ == "DegenerateInputError", kind
            with pytest.raises(H.DegenerateInputError):
                H.convex_hull_3d(pts)
            continue
        r = H.convex_hull_3d(pts)
        assert r.stats.perturbed == exp.perturbed, kind
        assert np.array_equal(r.faces, exp.faces), kind
        assert np.array_equal(r.vertices, exp.vertices), kind

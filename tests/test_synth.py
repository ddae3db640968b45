"""The seeded generators: determinism and the input-graph guarantees the oracle's
cheaper modes rely on (SURVEY Lemma L3: symmetrised K-NN ⊇ Čech)."""
import numpy as np

import pf_synth


def test_deterministic():
    a = pf_synth.make_scene("small", num_cells=800)
    b = pf_synth.make_scene("small", num_cells=800)
    for f in ("sites", "weights", "radii", "density", "rgb", "nbr_offsets", "nbr_indices"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_lists_are_exact_cech_complex():
    sc = pf_synth.make_scene("small", num_cells=1200)
    P = sc.sites.astype(np.float64)
    r = sc.radii.astype(np.float64)
    D = np.linalg.norm(P[:, None] - P[None], axis=-1)
    cech = (D < r[:, None] + r[None]) & ~np.eye(sc.num_cells, dtype=bool)
    got = np.zeros_like(cech)
    for i in range(sc.num_cells):
        got[i, sc.nbr_indices[sc.nbr_offsets[i]:sc.nbr_offsets[i + 1]]] = True
    assert np.array_equal(cech, got)
    assert np.array_equal(got, got.T)        # symmetric, no self loops
    assert np.all(sc.weights == sc.radii * sc.radii)


def test_tiny_sym8_contains_cech():
    sc = pf_synth.make_scene("tiny")
    P = sc.sites.astype(np.float64); r = sc.radii.astype(np.float64)
    for i in range(sc.num_cells):
        nb = set(sc.nbr_indices[sc.nbr_offsets[i]:sc.nbr_offsets[i + 1]].tolist())
        for j in range(sc.num_cells):
            if j != i and np.linalg.norm(P[i] - P[j]) < r[i] + r[j]:
                assert j in nb


def test_unfiltered_knn_variant_contains_cech_lists():
    """variant="knn" (bench --lists knn, the P:236 extraneous-edge comparison): same
    scene, lists = unfiltered sym-16NN, a strict superset of the Čech lists (Lemma L3)."""
    a = pf_synth.make_scene("small", num_cells=1500)
    b = pf_synth.make_scene("small", num_cells=1500, variant="knn")
    for f in ("sites", "weights", "radii", "density", "rgb"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert b.num_edges > 1.3 * a.num_edges
    for i in range(a.num_cells):
        ca = set(a.nbr_indices[a.nbr_offsets[i]:a.nbr_offsets[i + 1]].tolist())
        cb = b.nbr_indices[b.nbr_offsets[i]:b.nbr_offsets[i + 1]].tolist()
        assert ca <= set(cb) and i not in cb and len(cb) == len(set(cb))

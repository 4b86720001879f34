"""CPU: the C restatement (oracle/slcs_oracle.c) is pinned to the reference.

Golden vectors in tests/golden/ were produced by the reference's own code
(tests/golden/make_golden.py).  Known answers are the ones the reference's
test suites assert (file:line cited per test).
"""
import json
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_vectors.npz"))
D = json.load(open(os.path.join(HERE, "golden", "reference_dags.json")))


@pytest.mark.parametrize("i", range(5))
def test_kernels_match_reference_vectors(i):
    a, b, img = G[f"k{i}_a"], G[f"k{i}_b"], G[f"k{i}_img"]
    assert np.array_equal(O.logical_not(a), G[f"k{i}_not"])
    assert np.array_equal(O.logical_and(a, b), G[f"k{i}_and"])
    assert np.array_equal(O.logical_or(a, b), G[f"k{i}_or"])
    assert np.array_equal(O.dilate(a), G[f"k{i}_dilate"])
    assert O.count_true(a) == int(G[f"k{i}_count"][0])
    for op in range(5):
        for n in (62258.0, 56360.5, 0.0, 70000.0):
            assert np.array_equal(O.threshold(op, img, n), G[f"k{i}_thr{op}_{int(n * 2)}"])


def test_ccl_matches_reference_pointer_jumping():
    for i in range(8):
        assert np.array_equal(O.flood_fill_label(G[f"ccl{i}_in"]), G[f"ccl{i}_out"])
    for i in range(3):
        assert np.array_equal(O.flood_fill_label(G[f"cclb{i}_in"]), G[f"cclb{i}_out"])
    assert np.array_equal(O.flood_fill_label(G["concave_in"]), G["concave_out"])


def test_reach_matches_reference():
    for i in range(8):
        t, u = G[f"reach{i}_t"], G[f"reach{i}_u"]
        assert np.array_equal(O.reach(t, u), G[f"reach{i}_out"])
        assert np.array_equal(O.reach_bfs(t, u), G[f"reach{i}_out"])


def test_synth_fixtures_match_reference_checksums():
    assert np.array_equal(O.blob_noise(64, 64, 7), G["blob_64_7"])
    cs = D["checksums"]
    for key, want in cs.items():
        if key.startswith("blob_"):
            dims, seed = key[5:].split("_")
            w, h = map(int, dims.split("x"))
            if w * h > 1 << 20:
                continue  # the 4096^2 checksum is checked by the slow test below
            assert f"{O.checksum(O.blob_noise(w, h, int(seed))):016x}" == want, key
    # SURVEY.md §8c records concave-corner 128^2 FNV-1a = 1babecd38d348d25
    assert cs["concave_128"] == "1babecd38d348d25"


def test_blob_noise_4096_checksum():
    want = D["checksums"]["blob_4096x4096_1"]
    assert f"{O.checksum(O.blob_noise(4096, 4096, 1)):016x}" == want


def test_whole_formula_outputs_match_reference_executor():
    img = G["seg_in"]
    hI = O.threshold(0, img, 62258)
    vI = O.threshold(0, img, 56360)
    assert np.array_equal(O.grow(hI, vI), G["seg_out"])
    a, b = hI, vI
    x = O.logical_and(a, O.logical_not(b))
    for _ in range(4):
        x = O.dilate(x)
    assert np.array_equal(O.reach(x, b), G["c1_out"])


# ---- known answers from the reference suites ------------------------------------
def test_kat_threshold_strictness():  # test_kernels.cpp:69-90
    img = np.array([[62257, 62258, 62259]], np.uint16)
    assert O.threshold(0, img, 62258).tolist() == [[0, 0, 1]]
    assert O.threshold(3, img, 62258).tolist() == [[1, 1, 0]]
    assert O.threshold(2, img, 70000).tolist() == [[1, 1, 1]]
    ramp = np.arange(64, dtype=np.uint16).reshape(1, 64) * 1000
    assert O.threshold(4, ramp, 56360.5).sum() == 0


def test_kat_ccl():  # test_ccl.cpp:152-173, 224-232, 276-292
    l = O.flood_fill_label(np.ones((3, 3), np.uint8))
    assert (l == 9).all()  # packLabel(2,2,3)
    L = np.zeros((5, 5), np.uint8)
    L[0, :] = 1
    L[:, 0] = 1
    l = O.flood_fill_label(L)
    assert (l[L == 1] == 4 * 5 + 0 + 1).all()  # packLabel(4,0,5)
    chk = np.fromfunction(lambda r, c: (r + c) % 2 == 0, (8, 8)).astype(np.uint8)
    assert (O.flood_fill_label(chk)[chk == 1] == 64).all()  # packLabel(7,7,8)


def test_kat_reach_row():  # test_reach.cpp:61-71
    t = np.array([[0, 0, 0, 0, 1]], np.uint8)
    u = np.array([[0, 0, 1, 1, 0]], np.uint8)
    assert O.reach(t, u).tolist() == [[0, 1, 1, 1, 1]]


def test_kat_interior_border():  # test_reach.cpp:119-131
    assert (O.interior(np.ones((5, 5), np.uint8)) == 1).all()
    sq = np.zeros((8, 8), np.uint8)
    sq[2:6, 2:6] = 1
    core = np.zeros((8, 8), np.uint8)
    core[3:5, 3:5] = 1
    assert np.array_equal(O.interior(sq), core)


def test_maxvol_definition():
    # new opcode: union of maximal components, ties kept
    m = np.zeros((6, 9), np.uint8)
    m[0:2, 0:2] = 1
    m[0:2, 6:8] = 1
    m[5, 0] = 1
    out = O.maxvol(m)
    exp = m.copy()
    exp[5, 0] = 0
    assert np.array_equal(out, exp)
    assert O.maxvol(np.zeros((4, 4), np.uint8)).sum() == 0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_library_agrees_with_restatement_on_fresh_cases():
    R = O.Reference(workers=2)
    rng = O.Rng(4242)
    for _ in range(10):
        w, h = 5 + rng.below(60), 5 + rng.below(60)
        a = O.random_mask(w, h, rng.unit(), rng)
        t = O.random_mask(w, h, 0.1, rng)
        assert np.array_equal(R.ccl_label(a), O.flood_fill_label(a))
        assert np.array_equal(R.reach(t, a), O.reach(t, a))
        assert np.array_equal(R.dilate(a), O.dilate(a))

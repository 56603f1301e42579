"""The CPU oracle (oracle/layered_ref.c) pinned against the reference's own outputs.

tests/golden/*.npz were written by tests/golden/make_golden.py from the unmodified
reference package.  The oracle restates the reference in C with libm transcendentals,
so FP64 values agree to a few ulp (numpy's SIMD expm1/log1p differ from libm by 1 ulp
on ~2% of inputs) and every decision is bit-exact.
"""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, MERGE_EXAMPLE_TOP_PAIR, TEST_BASE_4x8_Z3, channel_llrs, load_code, make_code

oracle = pytest.importorskip("oracle.oracle")


def relerr(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


def test_oracle_phi_matches_reference():
    g = np.load(GOLDEN / "phi.npz")
    got = oracle.phi(g["x"])
    assert np.max(np.abs(got - g["phi"]) / g["phi"]) < 1e-14


def golden_code(name):
    if name == "t4x8z3":
        return make_code(TEST_BASE_4x8_Z3, 3, merged=False)
    if name == "merge3x3z5":
        return make_code(MERGE_EXAMPLE_TOP_PAIR, 5, merged=True)
    if name == "demo4x8z100":
        return load_code("demo_4x8_z100")
    return load_code("standin_v2_z100")


@pytest.mark.parametrize("name", ["t4x8z3", "merge3x3z5", "demo4x8z100", "standin_z100"])
def test_oracle_layers_match_reference(name):
    g = np.load(GOLDEN / f"layers_{name}.npz")
    base, sched, index = golden_code(name)
    code = oracle.OracleCode(index, sched)
    post = np.clip(g["llr"], -30, 30)
    assert np.array_equal(post, g["init_post"])
    msg = np.zeros((post.shape[0], index.total_edges * base.z))
    oracle.layer_update(code, 0, post, msg, g["syndrome"])
    assert relerr(post, g["l0_post"]) < 1e-13 and relerr(msg, g["l0_msg"]) < 1e-13
    for layer in range(1, len(sched.layers)):
        oracle.layer_update(code, layer, post, msg, g["syndrome"])
    assert relerr(post, g["sweep1_post"]) < 1e-12 and relerr(msg, g["sweep1_msg"]) < 1e-12
    for _ in range(4):
        oracle.layer_update(code, -1, post, msg, g["syndrome"])
    assert relerr(post, g["sweep5_post"]) < 1e-10
    assert np.array_equal(post < 0, g["sweep5_post"] < 0)


@pytest.mark.parametrize(
    "tag",
    [
        "decode_demo4x8z100_snr1_it10_noet",
        "decode_demo4x8z100_snr1_it10_et",
        "decode_demo4x8z100_snr2.5_it10_noet",
        "decode_demo4x8z100_snr2.5_it10_et",
        "decode_standin_z100_snr0.161_it10_noet",
        "decode_standin_z100_snr0.161_it50_noet",
        "decode_standin_z100_snr0.161_it50_et",
        "decode_standin_z100_snr0.2_it50_noet",
        "decode_standin_z100_snr0.2_it50_et",
    ],
)
def test_oracle_decode_matches_reference(tag):
    g = np.load(GOLDEN / f"{tag}.npz")
    name = "demo_4x8_z100" if "demo" in tag else "standin_v2_z100"
    base, sched, index = load_code(name)
    n = base.n_cols * base.z
    llr = channel_llrs(n, float(g["snr"]), int(g["seed"]), int(g["snr_idx"]), int(g["batch"]))
    assert hashlib.sha256(llr.tobytes()).hexdigest() == str(g["llr_sha"])
    code = oracle.OracleCode(index, sched)
    w, c, it, post = oracle.decode(code, llr, None, int(g["iters"]), bool(g["et"]), want_posterior=True)
    assert np.array_equal(c, g["converged"]) and np.array_equal(it, g["iterations"])
    assert np.array_equal(w, np.unpackbits(g["words"], axis=1)[:, :n])
    if "posterior" in g.files:
        assert relerr(post[:4], g["posterior"]) < 1e-8


def test_oracle_full_size_three_iterations():
    g = np.load(GOLDEN / "decode_standin_z2500_snr0.161_it3_noet.npz")
    base, sched, index = load_code("standin_v2_z2500")
    n = base.n_cols * base.z
    llr = channel_llrs(n, 0.161, 0, 0, 2)
    assert hashlib.sha256(llr.tobytes()).hexdigest() == str(g["llr_sha"])
    code = oracle.OracleCode(index, sched)
    w, c, it, post = oracle.decode(code, llr, None, 3, False, want_posterior=True)
    assert np.array_equal(w, np.unpackbits(g["words"], axis=1)[:, :n])
    assert relerr(post[:, g["sample_idx"]], g["sample_post"]) < 1e-11


def test_oracle_syndrome_matches_expansion():
    import paper_2004_09084_b200 as q

    rng = np.random.default_rng(5)
    base, sched, index = make_code(TEST_BASE_4x8_Z3, 3, merged=True)
    code = oracle.OracleCode(index, sched)
    words = rng.integers(0, 2, size=(4, 24)).astype(np.uint8)
    assert np.array_equal(oracle.syndrome(code, words), q.syndrome_of(words, q.expand(base)))

"""Parity of the CUDA path with the reference (golden fixtures) and the C oracle.

All tests here run on a B200 (``-m gpu``) and go through the C ABI.  Tolerances are
stated next to each assertion:
  * FP64 path (reference formula and fold order): posteriors/messages within 1e-12
    relative (|d| / max(|ref|, 1)) after a layer, 1e-10 after five sweeps -- the only
    differences are 1-ulp differences between libdevice and numpy's SIMD
    log1p/expm1; hard decisions, convergence flags and
    iteration counts bit-exact.
  * FP32 path: one layer / one sweep within 2e-5, five sweeps within 1e-4
    (north-star tolerance); hard decisions bit-exact after short decodes and after
    50 no-ET iterations in the pre-convergence regime (SNR 0.161); only no-ET decodes
    that run on past convergence into the clip-saturation regime (SNR 0.2) are
    compared by frame-level outcome.
"""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, channel_llrs, load_code, make_code, random_base_matrix

pytestmark = pytest.mark.gpu

TOL_LAYER = {"fp64": 1e-12, "fp32": 2e-5}
TOL_SWEEP5 = {"fp64": 1e-10, "fp32": 1e-4}


def relerr(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


def fresh_state(index, sched, batch, precision, engine=0):
    from paper_2004_09084_b200 import _native

    plan = _native.Plan(index, sched, 0)
    st = _native.State(plan, batch, precision)
    st.set_engine(engine)
    return plan, st


# ---------------------------------------------------------------------------- phi


@pytest.mark.parametrize("precision,tol", [("fp64", 4e-16 * 8), ("fp32", 3e-6)])
def test_device_phi(gpu, precision, tol):
    import paper_2004_09084_b200 as q

    g = np.load(GOLDEN / "phi.npz")
    got = q.phi(g["x"], precision=precision)
    x32 = g["x"].astype(np.float32).astype(np.float64)
    ref = g["phi"]
    if precision == "fp32":
        # compare against the exact function at the FP32-rounded argument
        ref = np.log1p(2.0 / np.expm1(np.clip(x32, 1e-10, 30.0)))
    rel = np.abs(got - ref) / ref
    assert np.isfinite(got).all() and (got > 0).all()
    assert rel.max() <= tol, rel.max()


def test_device_phi_clamps(gpu):
    import paper_2004_09084_b200 as q

    for precision in ("fp64", "fp32"):
        lo = q.phi(np.array([0.0, 1e-300, 1e-10]), precision=precision)
        hi = q.phi(np.array([30.0, 1e6]), precision=precision)
        assert lo[0] == lo[1] == lo[2] and hi[0] == hi[1]


# ---------------------------------------------------------------------- layers

LAYER_CASES = ["t4x8z3", "merge3x3z5", "demo4x8z100", "standin_z100"]


def golden_code(name):
    from conftest import MERGE_EXAMPLE_TOP_PAIR, TEST_BASE_4x8_Z3

    if name == "t4x8z3":
        return make_code(TEST_BASE_4x8_Z3, 3, merged=False)
    if name == "merge3x3z5":
        return make_code(MERGE_EXAMPLE_TOP_PAIR, 5, merged=True)
    if name == "demo4x8z100":
        return load_code("demo_4x8_z100")
    return load_code("standin_v2_z100")


@pytest.mark.parametrize("engine", [0, 1, 4])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", LAYER_CASES)
def test_layer_and_sweeps_match_reference(gpu, name, precision, engine):
    g = np.load(GOLDEN / f"layers_{name}.npz")
    base, sched, index = golden_code(name)
    assert np.array_equal(g["layers"], [len(l) for l in sched.layers])
    batch = g["llr"].shape[0]
    _, st = fresh_state(index, sched, batch, precision, engine)
    st.set_llr(g["llr"])
    st.reset(30.0)
    post, msg = st.download()
    assert np.array_equal(post, g["init_post"]) or precision == "fp32"
    assert relerr(post, g["init_post"]) <= 1e-7
    assert not msg.any()
    st.set_syndrome(g["syndrome"])
    st.layers(0, 1, 30.0, 1e-10)
    post, msg = st.download()
    assert relerr(post, g["l0_post"]) <= TOL_LAYER[precision]
    assert relerr(msg, g["l0_msg"]) <= TOL_LAYER[precision]
    # rest of the first sweep (includes the ragged merged layers of the stand-in)
    st.layers(1, len(sched.layers) - 1, 30.0, 1e-10)
    post, msg = st.download()
    assert relerr(post, g["sweep1_post"]) <= TOL_LAYER[precision] * 10
    assert relerr(msg, g["sweep1_msg"]) <= TOL_LAYER[precision] * 10
    for _ in range(4):
        st.layers(0, len(sched.layers), 30.0, 1e-10)
    post, _ = st.download()
    assert relerr(post, g["sweep5_post"]) <= TOL_SWEEP5[precision]
    # decisions bit-exact wherever the reference posterior is not within the stated
    # tolerance of zero (fp64: everywhere)
    ref = g["sweep5_post"]
    decided = np.abs(ref) > TOL_SWEEP5[precision] * np.maximum(np.abs(ref), 1.0)
    assert np.array_equal((post < 0)[decided], (ref < 0)[decided])


@pytest.mark.parametrize("batch", [2, 4, 8])
@pytest.mark.parametrize("engine", [0, 1, 4])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_layer_from_reference_state_with_messages(gpu, precision, engine, batch):
    """One layer from a mid-decode reference state (nonzero messages), per layer.

    Batches 2/4/8 give lane widths W = 2/4/8, i.e. both the direct kernel and the
    TMA pipeline (bulk copies need W * sizeof(T) to be a multiple of 16 bytes)."""
    from oracle import oracle

    g = np.load(GOLDEN / "layers_standin_z100.npz")
    base, sched, index = load_code("standin_v2_z100")
    code = oracle.OracleCode(index, sched)
    reps = batch // g["llr"].shape[0]
    gsyn = np.tile(g["syndrome"], (reps, 1))
    gpost, gmsg = np.tile(g["sweep1_post"], (reps, 1)), np.tile(g["sweep1_msg"], (reps, 1))
    _, st = fresh_state(index, sched, batch, precision, engine)
    st.set_syndrome(gsyn)
    for layer in range(len(sched.layers)):
        post = gpost.copy()
        msg = gmsg.copy()
        st.upload(post, msg)
        st.layers(layer, 1, 30.0, 1e-10)
        dpost, dmsg = st.download()
        oracle.layer_update(code, layer, post, msg, gsyn)
        assert relerr(dpost, post) <= TOL_LAYER[precision], layer
        assert relerr(dmsg, msg) <= TOL_LAYER[precision], layer


# ---------------------------------------------------------------------- decodes

DECODE_CASES = [
    "decode_demo4x8z100_snr1_it10_noet",
    "decode_demo4x8z100_snr1_it10_et",
    "decode_demo4x8z100_snr2.5_it10_noet",
    "decode_demo4x8z100_snr2.5_it10_et",
    "decode_standin_z100_snr0.161_it10_noet",
    "decode_standin_z100_snr0.161_it50_noet",
    "decode_standin_z100_snr0.161_it50_et",
    "decode_standin_z100_snr0.2_it50_noet",
    "decode_standin_z100_snr0.2_it50_et",
]


def run_golden_decode(tag, precision):
    import paper_2004_09084_b200 as q

    g = np.load(GOLDEN / f"{tag}.npz")
    name = "demo_4x8_z100" if "demo" in tag else "standin_v2_z100"
    base, sched, index = load_code(name)
    n, m = base.n_cols * base.z, base.n_rows * base.z
    batch = int(g["batch"])
    llr = channel_llrs(n, float(g["snr"]), int(g["seed"]), int(g["snr_idx"]), batch)
    assert hashlib.sha256(llr.tobytes()).hexdigest() == str(g["llr_sha"])  # host channel mirror bit-exact
    cfg = q.DecoderConfig(max_iterations=int(g["iters"]), early_termination=bool(g["et"]))
    dec = q.LayeredDecoder(index, sched, cfg, precision=precision)
    w, c, it = dec.decode_batch_arrays(llr, np.zeros((batch, m), np.uint8))
    ref_w = np.unpackbits(g["words"], axis=1)[:, :n]
    return g, w, c, it, ref_w


@pytest.mark.parametrize("tag", DECODE_CASES)
def test_decode_fp64_bit_exact(gpu, tag):
    g, w, c, it, ref_w = run_golden_decode(tag, "fp64")
    assert np.array_equal(c, g["converged"])
    assert np.array_equal(it, g["iterations"])
    assert int((w != ref_w).sum()) == 0


@pytest.mark.parametrize("tag", DECODE_CASES)
def test_decode_fp32_against_reference(gpu, tag):
    """FP32 contract, by regime:
      * early-termination runs and 10-iteration runs: converged flags and iteration
        counts identical, hard decisions bit-exact (every converged frame, every frame
        of the 10-iteration runs);
      * 50 no-ET iterations at SNR 0.161 (pre-convergence): flags and iterations
        identical, hard decisions identical wherever the reference posterior satisfies
        |L| >= 1e-3 (the FP32 margin of tests/test_bench_config_parity.py);
      * 50 no-ET iterations at SNR 0.2 (frames converge and then keep iterating into
        the LLR-clip saturation regime): FP32 and FP64 trajectories
        separate chaotically after convergence, so only the frame-level outcome is
        compared -- convergence flags agree on >= 75% of frames; bit mismatches are
        reported."""
    g, w, c, it, ref_w = run_golden_decode(tag, "fp32")
    ref_c = g["converged"]
    flips = int((w != ref_w).sum())
    frames_differ = int((w != ref_w).any(axis=1).sum())
    print(f"{tag}: fp32 bit mismatches {flips} in {frames_differ} frames; "
          f"converged {int(c.sum())} vs reference {int(ref_c.sum())}")
    if bool(g["et"]):
        assert np.array_equal(c, ref_c) and np.array_equal(it, g["iterations"])
        assert np.array_equal(w[ref_c], ref_w[ref_c])
    elif "it10" in tag:
        assert np.array_equal(c, ref_c) and np.array_equal(it, g["iterations"])
        assert flips == 0
    elif "snr0.161" in tag:
        # 50 iterations amplify the FP32 state's rounding (tests/test_bench_config_parity.py):
        # decisions identical wherever the reference posterior is not within 1e-3 of zero
        assert np.array_equal(c, ref_c) and np.array_equal(it, g["iterations"])
        from oracle import oracle

        base, sched, index = load_code("standin_v2_z100")
        llr = channel_llrs(base.n_cols * base.z, float(g["snr"]), int(g["seed"]), int(g["snr_idx"]), len(c))
        ow, _, _, opost = oracle.decode(oracle.OracleCode(index, sched), llr, None, int(g["iters"]), False,
                                        want_posterior=True)
        assert np.array_equal(ow, ref_w)  # the oracle reproduces the reference's decisions
        margin = np.abs(opost[w != ref_w])
        print(f"{tag}: reference |L| at the flips {np.sort(margin).tolist()}")
        assert (margin < 1e-3).all()
    else:
        assert (c == ref_c).mean() >= 0.75


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_posterior_after_decode(gpu, precision):
    """Posterior after 10 and 50 sweeps (SNR 0.161, z=100 twin) vs the reference."""
    for tag, tol in [("decode_standin_z100_snr0.161_it10_noet", {"fp64": 1e-9, "fp32": 1e-4}),
                     ("decode_standin_z100_snr0.161_it50_noet", {"fp64": 1e-6, "fp32": 1e-3})]:
        g = np.load(GOLDEN / f"{tag}.npz")
        base, sched, index = load_code("standin_v2_z100")
        n = base.n_cols * base.z
        llr = channel_llrs(n, float(g["snr"]), int(g["seed"]), int(g["snr_idx"]), 4)
        _, st = fresh_state(index, sched, 4, precision)
        st.set_llr(llr)
        st.reset(30.0)
        st.set_syndrome(None)
        for _ in range(int(g["iters"])):
            st.layers(0, len(sched.layers), 30.0, 1e-10)
        post, _ = st.download()
        err = relerr(post, g["posterior"])
        print(f"{tag} {precision}: max rel posterior error {err:.3g}")
        assert err <= tol[precision]


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_full_size_code_three_iterations(gpu, precision):
    """n = 10^6 stand-in (z=2500), 2 frames, 3 iterations: decisions and sampled posteriors."""
    import paper_2004_09084_b200 as q

    g = np.load(GOLDEN / "decode_standin_z2500_snr0.161_it3_noet.npz")
    base, sched, index = load_code("standin_v2_z2500")
    n = base.n_cols * base.z
    llr = channel_llrs(n, 0.161, 0, 0, 2)
    assert hashlib.sha256(llr.tobytes()).hexdigest() == str(g["llr_sha"])
    _, st = fresh_state(index, sched, 2, precision)
    st.set_llr(llr)
    st.reset(30.0)
    st.set_syndrome(None)
    for _ in range(3):
        st.layers(0, len(sched.layers), 30.0, 1e-10)
    post, _ = st.download()
    ref_w = np.unpackbits(g["words"], axis=1)[:, :n]
    assert np.array_equal((post < 0).astype(np.uint8), ref_w)
    assert relerr(post[:, g["sample_idx"]], g["sample_post"]) <= {"fp64": 1e-11, "fp32": 2e-5}[precision]
    # the decode entry point agrees with the state path
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=3, early_termination=False),
                           precision=precision)
    w, c, it = dec.decode_batch_arrays(llr, np.zeros((2, base.n_rows * base.z), np.uint8))
    assert np.array_equal(w, ref_w) and (it == 3).all()


# ------------------------------------------------------------ random codes vs oracle


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_random_codes_against_oracle(gpu, precision):
    """100 random codes (degrees 1..12, z 1..16), random syndromes, B in {1,3,5}."""
    import paper_2004_09084_b200 as q
    from oracle import oracle

    rng = np.random.default_rng(20240901)
    for trial in range(100):
        shifts, z = random_base_matrix(rng)
        merged = bool(trial % 2)
        base, sched, index = make_code(shifts, z, merged=merged)
        code = oracle.OracleCode(index, sched)
        batch = (1, 3, 5)[trial % 3]
        n, m = base.n_cols * z, base.n_rows * z
        llr = rng.normal(0.5, 2.0, size=(batch, n))
        syn = (rng.random((batch, m)) < 0.3).astype(np.uint8)
        # one sweep, state parity
        _, st = fresh_state(index, sched, batch, precision)
        post = np.clip(llr, -30, 30)
        msg = np.zeros((batch, index.total_edges * z))
        st.upload(post, msg)
        st.set_syndrome(syn)
        st.layers(0, len(sched.layers), 30.0, 1e-10)
        dpost, dmsg = st.download()
        oracle.layer_update(code, -1, post, msg, syn)
        assert relerr(dpost, post) <= TOL_LAYER[precision] * 10, trial
        assert relerr(dmsg, msg) <= TOL_LAYER[precision] * 10, trial
        # full decode with ET: outcomes
        if precision == "fp64":
            ow, oc, oi = oracle.decode(code, llr, syn, 20, True)
            dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=20), precision=precision)
            w, c, it = dec.decode_batch_arrays(llr, syn)
            assert np.array_equal(c, oc) and np.array_equal(it, oi), trial
            assert np.array_equal(w, ow), trial


def test_wide_rows_fp64_against_oracle(gpu):
    """Row degrees 13..24 (the per-layer engines' wide buckets; FP64 rows above 16 run on
    the direct kernel): FP64 decodes bit-exact against the C oracle, FP32 sweeps close."""
    import paper_2004_09084_b200 as q
    from oracle import oracle

    rng = np.random.default_rng(5)
    for trial in range(8):
        n_rows, n_cols, z = int(rng.integers(1, 4)), 26, int(rng.integers(2, 12))
        shifts = np.full((n_rows, n_cols), -1, dtype=np.int64)
        for i in range(n_rows):
            deg = int(rng.integers(13, 25))
            cols = rng.choice(n_cols, size=deg, replace=False)
            shifts[i, cols] = rng.integers(0, z, size=deg)
        base, sched, index = make_code(shifts.tolist(), z, merged=bool(trial % 2))
        code = oracle.OracleCode(index, sched)
        batch = (2, 5, 9)[trial % 3]
        n, m = base.n_cols * z, base.n_rows * z
        llr = rng.normal(1.0, 2.0, size=(batch, n))
        syn = (rng.random((batch, m)) < 0.3).astype(np.uint8)
        ow, oc, oi = oracle.decode(code, llr, syn, 12, True)
        w, c, it = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=12),
                                    precision="fp64").decode_batch_arrays(llr, syn)
        assert np.array_equal(c, oc) and np.array_equal(it, oi) and np.array_equal(w, ow), trial
        _, st = fresh_state(index, sched, batch, "fp32")
        post = np.clip(llr, -30, 30)
        msg = np.zeros((batch, index.total_edges * z))
        st.upload(post, msg)
        st.set_syndrome(syn)
        st.layers(0, len(sched.layers), 30.0, 1e-10)
        dpost, dmsg = st.download()
        oracle.layer_update(code, -1, post, msg, syn)
        assert relerr(dpost, post) <= TOL_LAYER["fp32"] * 10 and relerr(dmsg, msg) <= TOL_LAYER["fp32"] * 10, trial


@pytest.mark.parametrize("batch", [1, 2, 3, 31, 33, 64, 70])
def test_batch_padding_and_lane_groups(gpu, batch):
    """Any batch size: lane groups are padded; results equal the oracle frame by frame."""
    import paper_2004_09084_b200 as q
    from oracle import oracle

    base, sched, index = load_code("demo_4x8_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, 1.6, 20240901, 3, batch)
    code = oracle.OracleCode(index, sched)
    ow, oc, oi = oracle.decode(code, llr, None, 30, True)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=30), precision="fp64")
    w, c, it = dec.decode_batch_arrays(llr, np.zeros((batch, m), np.uint8))
    assert np.array_equal(c, oc) and np.array_equal(it, oi) and np.array_equal(w, ow)


def test_adversarial_llrs_stay_clipped(gpu):
    """+-inf, 1e308, -0.0, denormals (test_decoder.py:168-203 analogue) on both paths."""
    from conftest import TEST_BASE_4x8_Z3

    base, sched, index = make_code(TEST_BASE_4x8_Z3, 3)
    llr = np.array([[np.inf, -np.inf, 0.0, -0.0, 1e-300, -5.0, 1e308, -1e308] * 3])
    syn = (np.arange(12) % 2).astype(np.uint8)[None]
    for precision in ("fp64", "fp32"):
        _, st = fresh_state(index, sched, 1, precision)
        st.set_llr(llr)
        st.reset(8.0)
        st.set_syndrome(syn)
        for _ in range(3):
            st.layers(0, len(sched.layers), 8.0, 1e-10)
            post, msg = st.download()
            assert np.isfinite(post).all() and np.abs(post).max() <= 8.0
            assert np.isfinite(msg).all() and np.abs(msg).max() <= 8.0


def test_negative_zero_hard_decision(gpu):
    """-0.0 decides to bit 0 (decoder.py:264-266, test_decoder.py:223-227)."""
    import paper_2004_09084_b200 as q

    base, sched, index = make_code([[0, 0]], 1)
    for precision in ("fp64", "fp32"):
        dec = q.LayeredDecoder(index, sched, q.DecoderConfig(), precision=precision)
        st = dec.new_state(np.array([0.0, -0.0]))
        assert dec.hard_decision(st).tolist() == [[0, 0]]


# ------------------------------------------------------------ device channel


def test_device_channel_statistics_and_sharding_invariance(gpu):
    """Philox BIAWGN: moments match N(2 snr, 4 snr); frames independent of batch offsets."""
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code("standin_v2_z100")
    plan = _native.Plan(index, sched, 0)
    snr = 0.161
    st = _native.State(plan, 8, "fp64")
    st.set_llr_synthetic(seed=5, snr_idx=2, first_frame=0, snr=snr)
    llr = st.get_llr()
    assert abs(llr.mean() - 2 * snr) < 0.01
    assert abs(llr.std() - np.sqrt(4 * snr)) < 0.01
    # frames 4..7 generated by a second "GPU" with first_frame=4 are identical
    st2 = _native.State(plan, 4, "fp64")
    st2.set_llr_synthetic(seed=5, snr_idx=2, first_frame=4, snr=snr)
    assert np.array_equal(st2.get_llr(), llr[4:])
    # fp32 state holds the same values rounded
    st3 = _native.State(plan, 8, "fp32")
    st3.set_llr_synthetic(seed=5, snr_idx=2, first_frame=0, snr=snr)
    assert np.array_equal(st3.get_llr(), llr.astype(np.float32).astype(np.float64))


def test_device_encode_mode_syndrome(gpu):
    """Encode mode: the device target syndrome equals H * truth (oracle), and a strong
    channel decodes to the truth (bench.py:216-228 encode_mode semantics)."""
    from oracle import oracle
    from paper_2004_09084_b200 import _native
    import paper_2004_09084_b200 as q

    base, sched, index = load_code("demo_4x8_z100")
    code = oracle.OracleCode(index, sched)
    plan = _native.Plan(index, sched, 0)
    st = _native.State(plan, 6, "fp32")
    st.set_llr_synthetic(seed=1, snr_idx=0, first_frame=0, snr=8.0, encode_mode=True)
    truths = st.truths()
    assert 0.4 < truths.mean() < 0.6
    qcfg = _native.make_config(q.DecoderConfig(max_iterations=20), "fp32")
    st.decode(qcfg)
    w, c, it = st.results()
    assert c.all() and np.array_equal(w, truths)
    # the syndrome the device targeted is H * truths
    assert np.array_equal(oracle.syndrome(code, w), oracle.syndrome(code, truths))


@pytest.mark.parametrize("precision", ["fp64", "fp32", "fp32-msg16"])
def test_decode_stream_matches_blocking_calls(gpu, precision):
    """decode_stream (async copies, double-buffered workspaces) == decode_batch_arrays,
    including nonzero syndromes, early termination and a batch-size change mid-stream."""
    import paper_2004_09084_b200 as q
    from conftest import TEST_BASE_4x8_Z3

    base, sched, index = load_code("demo_4x8_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    rows = q.expand(base)
    rng = np.random.default_rng(11)
    batches = []
    for i, bsz in enumerate([8, 8, 5, 8]):
        words = rng.integers(0, 2, size=(bsz, n)).astype(np.uint8) if i % 2 else np.zeros((bsz, n), np.uint8)
        llr = (1.0 - 2.0 * words) * 2.5 + rng.normal(0, 1.2, size=(bsz, n))
        batches.append((llr, q.syndrome_of(words, rows)))
    for et in (True, False):
        cfg = q.DecoderConfig(max_iterations=20, early_termination=et)
        dec = q.LayeredDecoder(index, sched, cfg, precision=precision)
        ref = [dec.decode_batch_arrays(l, s) for l, s in batches]
        got = list(dec.decode_stream(batches, depth=2, copy=True))
        for (w0, c0, i0), (w1, c1, i1) in zip(ref, got):
            assert np.array_equal(w0, w1) and np.array_equal(c0, c1) and np.array_equal(i0, i1)


def test_device_channel_distribution(gpu):
    """Philox BIAWGN beyond its moments (round-1 review): 8 M device LLRs of the all-zero
    word at SNR 0.161 against N(2 snr, 4 snr) -- Kolmogorov-Smirnov distance, tail masses
    at 3/4/5 sigma within Poisson bounds of the Gaussian's, lag-1 correlation along a
    frame and between frames ~0.  Box-Muller on 32-bit uniforms cannot go beyond
    sqrt(-2 ln 2^-32) = 6.66 sigma (expected count beyond that at 8 M draws: 2e-4)."""
    from scipy import stats

    from paper_2004_09084_b200 import _native

    base, sched, index = load_code("standin_v2_z2500")
    snr = 0.161
    st = _native.State(_native.Plan(index, sched, 0), 8, "fp64")
    st.set_llr_synthetic(seed=11, snr_idx=3, first_frame=0, snr=snr)
    llr = st.get_llr()
    z = ((llr - 2 * snr) / np.sqrt(4 * snr)).reshape(-1)
    ks = stats.kstest(z, "norm")
    assert ks.statistic < 1e-3 and ks.pvalue > 1e-4, ks
    for k in (3.0, 4.0, 5.0):
        observed = int((np.abs(z) > k).sum())
        expected = z.size * 2 * stats.norm.sf(k)
        assert abs(observed - expected) <= 5 * np.sqrt(expected) + 2, (k, observed, expected)
    assert np.abs(z).max() < 6.7
    assert abs(np.corrcoef(z[:-1], z[1:])[0, 1]) < 2e-3
    f = z.reshape(8, -1)
    assert np.abs(np.corrcoef(f)[np.triu_indices(8, 1)]).max() < 5e-3


def test_pageable_and_pinned_host_buffers_agree(gpu):
    """The host staging pipeline (csrc/hostio.h): 16 codewords of the n = 10^6 code as
    pageable float64 (the reference's format; 128 MB through the 8 MB pinned ring, converted
    to float32 on the host threads), pageable float32, and pinned float32, with a nonzero
    target syndrome -- identical outcomes; words read back through the ring into pageable
    memory (16 MB, two chunks) equal the pinned path's."""
    import paper_2004_09084_b200 as q
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code("standin_v2_z2500")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    rng = np.random.default_rng(5)
    llr = rng.normal(3.0, 2.0, size=(16, n))
    syn = (rng.random((16, m)) < 0.001).astype(np.uint8)
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=3, early_termination=False))
    a = dec.decode_batch_arrays(llr, syn)
    b = dec.decode_batch_arrays(llr.astype(np.float32), syn)
    pin = _native.PinnedArray((16, n), np.float32)
    pin.array[...] = llr
    spin = _native.PinnedArray((16, m), np.uint8)
    spin.array[...] = syn
    c = dec.decode_batch_arrays(pin.array, spin.array)
    for x, y, z in zip(a, b, c):
        assert np.array_equal(x, y) and np.array_equal(x, z)
    assert a[0].any() and not a[0].all()


def test_stream_results_outlive_their_slots(gpu):
    """a yielded words array is a view of a pinned slot buffer; dropping the
    decoder's slots (a batch-size or depth change) must not free memory a view still uses."""
    import gc

    import paper_2004_09084_b200 as q

    base, sched, index = load_code("demo_4x8_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = np.random.default_rng(2).normal(2.0, 1.0, size=(8, n))
    dec = q.LayeredDecoder(index, sched, q.DecoderConfig(max_iterations=5, early_termination=False))
    kept = [w for w, _, _ in dec.decode_stream([(llr, np.zeros((8, m), np.uint8))], depth=1)]
    snapshot = kept[0].copy()
    list(dec.decode_stream([(llr[:3], np.zeros((3, m), np.uint8))], depth=2))  # replaces the slot cache
    dec = None
    gc.collect()
    assert np.array_equal(kept[0], snapshot)


def test_wait_covers_uploads_without_a_decode(gpu):
    """qcl_state_wait blocks for everything queued on the state (here only the staged LLR
    upload) and reports 0 ms when no decode was queued (it used to fail on the unrecorded
    timing events)."""
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code("demo_4x8_z100")
    n = base.n_cols * base.z
    st = _native.State(_native.Plan(index, sched, 0), 4, "fp32")
    llr = np.random.default_rng(5).normal(1.0, 2.0, size=(4, n))
    st.set_llr(llr)
    assert st.wait() == 0.0
    assert np.array_equal(st.get_llr(), llr.astype(np.float32).astype(np.float64))

"""Opt-in FP16 edge messages (``precision="fp32-msg16"``, QCL_PREC_FP32_MSG16; SURVEY §8f
row 4, the "beyond-parity modes" of the paper's message packing).

Posteriors stay FP32; every new message |r| is rounded to FP16 before it updates the
posterior and is stored, so a sweep's q = L - r_old subtracts exactly what the previous
sweep added.  This mode is NOT bit-identical to the FP32 path, so parity here is:
  * per sweep: posteriors and messages within the FP16 rounding of |r| <= clip (tolerances
    written below) of the FP32 flow engine on the same state;
  * per campaign: FER inside the reference acceptance CI (test_acceptance.py:194,236) of
    the FP32 path on the same device-channel frames;
  * the state it stores really is FP16 (download == FP16 rounding of an upload).
"""

import math

import numpy as np
import pytest

from conftest import ROOT, channel_llrs, load_code


def test_precision_code_matches_header():
    from paper_2004_09084_b200 import _native

    header = (ROOT / "include" / "qcldpc_b200.h").read_text()
    assert "#define QCL_PREC_FP32_MSG16 2" in header
    assert _native.PREC["fp32-msg16"] == 2


def test_decoder_and_campaign_accept_the_precision():
    from paper_2004_09084_b200.campaign import CampaignConfig

    CampaignConfig(matrix_path=str(ROOT / "codes" / "demo_4x8_z100.txt"), snr_list=(1.0,), precision="fp32-msg16")
    with pytest.raises(ValueError):
        CampaignConfig(matrix_path=str(ROOT / "codes" / "demo_4x8_z100.txt"), snr_list=(1.0,), precision="fp8")


def _state(plan, batch, precision, llr, syn=None):
    from paper_2004_09084_b200 import _native

    st = _native.State(plan, batch, precision)
    st.set_llr(llr)
    st.reset(30.0)
    st.set_syndrome(syn)
    return st


@pytest.mark.gpu
def test_upload_download_rounds_messages_to_fp16(gpu):
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code("standin_v2_z100")
    plan = _native.Plan(index, sched, 0)
    n = base.n_cols * base.z
    st = _native.State(plan, 8, "fp32-msg16")
    _, msg0 = st.download()
    ez = msg0.shape[1]
    rng = np.random.default_rng(0)
    post = rng.normal(0, 5, size=(8, n))
    msg = rng.normal(0, 5, size=(8, ez))
    st.upload(post, msg)
    got_post, got_msg = st.download()
    assert np.array_equal(got_post, post.astype(np.float32).astype(np.float64))
    assert np.array_equal(got_msg, msg.astype(np.float16).astype(np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("name,batch,sweeps,syn", [("standin_v2_z100", 16, 1, False), ("standin_v2_z100", 64, 3, False),
                                                   ("demo_6x12_z16", 33, 2, False), ("standin_v2_z2500", 8, 1, False),
                                                   ("standin_v2_z100", 16, 2, True), ("demo_6x12_z16", 33, 2, True)])
def test_sweeps_within_fp16_rounding_of_fp32(gpu, name, batch, sweeps, syn):
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code(name)
    plan = _native.Plan(index, sched, 0)
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, 0.5, seed=1, snr_idx=0, frames=batch)
    target = (np.random.default_rng(2).random((batch, m)) < 0.5).astype(np.uint8) if syn else None
    a = _state(plan, batch, "fp32", llr, target)
    b = _state(plan, batch, "fp32-msg16", llr, target)
    for _ in range(sweeps):
        for st in (a, b):
            st.layers(0, len(sched.layers), 30.0, 1e-10)
    (la, ra), (lb, rb) = a.download(), b.download()
    # every stored message is an FP16 value
    assert np.array_equal(rb, rb.astype(np.float16).astype(np.float64))
    # Each new |r| is off by its FP16 rounding (<= 2^-11 |r|), and within a sweep later
    # layers see the posteriors those errors moved.  Measured on B200 (tools/msg16_diag.py):
    # max |dL| = max |dR| = 0.008-0.009 after one sweep, 0.023 after three (zero target),
    # 0.032 after two with a random target syndrome; mean |dL| 1e-4..6e-4 (2e-3 with the
    # random target); sign flips 0..2.6e-5 of the posteriors (near-zero values at SNR 0.5),
    # 2.8e-4 with a random target (many posteriors near zero; 1 of 6336 on the 192-bit code).
    tol = 0.02 * sweeps ** 2
    assert np.max(np.abs(lb - la)) <= tol and np.max(np.abs(rb - ra)) <= tol
    assert np.mean(np.abs(lb - la)) <= 2e-3 * sweeps and np.mean(np.abs(rb - ra)) <= 2e-3 * sweeps
    flips = np.count_nonzero((la < 0) != (lb < 0))
    assert flips <= max(2, (5e-4 if syn else 1e-4) * la.size), flips


@pytest.mark.gpu
def test_decodes_match_fp32_outcomes_statistically(gpu):
    import paper_2004_09084_b200 as q

    base, sched, index = load_code("standin_v2_z100")
    n, m = base.n_cols * base.z, base.n_rows * base.z
    llr = channel_llrs(n, 0.2, seed=0, snr_idx=0, frames=64)
    cfg = q.DecoderConfig(max_iterations=50, early_termination=True)
    res = {}
    for prec in ("fp32", "fp32-msg16"):
        dec = q.LayeredDecoder(index, sched, cfg, precision=prec)
        res[prec] = dec.decode_batch_arrays(llr, np.zeros((64, m), np.uint8))
    (wa, ca, ia), (wb, cb, ib) = res["fp32"], res["fp32-msg16"]
    assert abs(int(ca.sum()) - int(cb.sum())) <= 2
    both = ca & cb
    assert np.array_equal(wa[both], wb[both])  # converged words are the codeword
    assert abs(float(ia.mean()) - float(ib.mean())) <= 0.5


@pytest.mark.gpu
def test_campaign_fer_within_ci_of_fp32(gpu):
    from paper_2004_09084_b200.campaign import CampaignConfig, run_campaign

    kw = dict(matrix_path=str(ROOT / "codes" / "standin_v2_z100.txt"), snr_list=(0.17, 0.2), max_iterations=40,
              early_termination=True, batch_size=64, min_trials=512, seed=7, channel="device")
    a = run_campaign(CampaignConfig(**kw, precision="fp32"))
    b = run_campaign(CampaignConfig(**kw, precision="fp32-msg16"))
    assert b.metadata["device"]["frame_pool"]
    for x, y in zip(a.cells, b.cells):
        band = 1.96 * math.sqrt(x.fer * (1 - x.fer) / 512 + y.fer * (1 - y.fer) / 512) + 1.0 / 512
        assert abs(x.fer - y.fer) <= band, (x, y)


@pytest.mark.gpu
def test_paths_without_fp16_messages_fail_loudly(gpu):
    from paper_2004_09084_b200 import _native

    base, sched, index = load_code("standin_v2_z100")
    plan = _native.Plan(index, sched, 0)
    st = _native.State(plan, 8, "fp32-msg16")
    st.reset(30.0)
    with pytest.raises(RuntimeError, match="flow engine"):
        st.layers(0, 1, 30.0, 1e-10)  # a single layer runs on the per-layer kernels
    with pytest.raises(RuntimeError, match="flow engine"):
        st.set_engine(0)

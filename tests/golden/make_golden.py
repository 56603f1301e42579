"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container, where the reference is importable read-only:

    python tests/golden/make_golden.py            # needs /root/reference/pkg/src

Every array written here is an output of the unmodified reference package
(``qcldpc`` from /root/reference/pkg/src): its phi, its layer updates, its sweeps and
its full decodes.  The fixtures pin the C oracle (tests/test_oracle.py, CPU) and the
CUDA path (tests/test_device_parity.py, GPU).  Nothing at test time reads
/root/reference; only these committed .npz/.txt files travel.

Cases (SURVEY.md section 8c "golden vectors to generate"):
  * phi on a log grid;
  * per-layer states (layer 0, the ragged layers, one full sweep, five sweeps) on
    TEST_BASE_4x8_Z3 (z=3), the merged 3x3 example (z=5), demo_4x8_z100 (config 1),
    and the z=100 twin of the rate-0.1 stand-in (ragged merged layers, degrees 4/10/11),
    with random nonzero syndromes;
  * full decodes: config 1 (B=64, SNR 1.0/2.5, 10 it, ET on/off), stand-in z=100
    (B=16, SNR 0.161 and 0.2, 50 it, ET on/off), stand-in z=2500 (B=2, 3 it, no ET);
  * host-channel checksums (frame_rng / transmit / init_llr) so the PCG64 mirror is
    pinned bit-exactly.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src")
REF_CODES = Path("/root/reference/pkg/codes")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))

import qcldpc  # noqa: E402  (the reference)
from qcldpc.channel import ChannelConfig, frame_rng, init_llr, transmit  # noqa: E402

from paper_2004_09084_b200.standin import standin_v2  # noqa: E402  (our generator; matrix only)

TEST_BASE_4x8_Z3 = [
    [0, 1, -1, -1, 2, -1, 1, -1],
    [0, -1, 1, -1, -1, 2, 0, -1],
    [-1, 2, -1, 0, -1, 1, -1, 2],
    [-1, -1, 2, 1, 0, -1, -1, 2],
]
MERGE_EXAMPLE_TOP_PAIR = [[1, -1, -1], [-1, 2, 1], [2, 0, 0]]


def ref_code(shifts, z, merged):
    base = qcldpc.BaseMatrix(len(shifts), len(shifts[0]), z, np.asarray(shifts))
    sched = qcldpc.greedy_schedule(base) if merged else qcldpc.single_row_schedule(base)
    return base, sched, qcldpc.build_compact_index(base, sched)


def write_codes():
    codes = ROOT / "codes"
    codes.mkdir(exist_ok=True)
    for name in ("demo_4x8_z32", "demo_4x8_z100", "demo_6x12_z16"):
        base = qcldpc.load_base_matrix(REF_CODES / f"{name}.txt")
        (codes / f"{name}.txt").write_text(qcldpc.serialize_base_matrix(base))
    for z in (100, 2500):
        ours = standin_v2(z=z)
        base = qcldpc.BaseMatrix(ours.n_rows, ours.n_cols, z, ours.shifts)
        (codes / f"standin_v2_z{z}.txt").write_text(qcldpc.serialize_base_matrix(base))


def channel_llrs(n, snr, seed, snr_idx, frames, start=0):
    chan = ChannelConfig(snr=snr, seed=seed)
    return np.stack(
        [init_llr(transmit(np.zeros(n, np.uint8), chan, frame_rng(seed, snr_idx, start + i)), chan) for i in range(frames)]
    )


def layer_case(name, base, sched, index, batch, snr, seed):
    z = base.z
    n, m = base.n_cols * z, base.n_rows * z
    rng = np.random.default_rng(seed)
    llr = channel_llrs(n, snr, seed, 0, batch)
    syn = (rng.random((batch, m)) < 0.5).astype(np.uint8)
    dec = qcldpc.LayeredDecoder(index, sched, qcldpc.DecoderConfig())
    out = dict(llr=llr, syndrome=syn, layers=np.array([len(l) for l in sched.layers]))
    st = dec.new_state(llr)
    out["init_post"] = st.posterior.copy()
    dec.layer_update(st, 0, syn)
    out["l0_post"], out["l0_msg"] = st.posterior.copy(), st.edge_messages.copy()
    # continue the sweep; record every layer's state (ragged layers included)
    for l in range(1, len(sched.layers)):
        dec.layer_update(st, l, syn)
    out["sweep1_post"], out["sweep1_msg"] = st.posterior.copy(), st.edge_messages.copy()
    for _ in range(4):
        dec._sweep(st, dec._check_syndrome(syn, batch))
    out["sweep5_post"] = st.posterior.copy()
    np.savez_compressed(HERE / f"layers_{name}.npz", **out)


def decode_case(name, base, sched, index, batch, snr, iters, et, seed=20240901, snr_idx=0, keep_post=False):
    z = base.z
    n, m = base.n_cols * z, base.n_rows * z
    llr = channel_llrs(n, snr, seed, snr_idx, batch)
    dec = qcldpc.LayeredDecoder(index, sched, qcldpc.DecoderConfig(max_iterations=iters, early_termination=et))
    words, conv, it = dec.decode_batch_arrays(llr, np.zeros((batch, m), np.uint8))
    out = dict(
        seed=seed, snr=snr, snr_idx=snr_idx, batch=batch, iters=iters, et=et,
        llr_sha=hashlib.sha256(llr.tobytes()).hexdigest(),
        words=np.packbits(words, axis=1), converged=conv, iterations=it,
    )
    if keep_post:
        st = dec.new_state(llr)
        syn = np.zeros((batch, m), bool)
        for _ in range(iters):
            dec._sweep(st, syn)
        out["posterior"] = st.posterior[:4].astype(np.float64)
    tag = f"decode_{name}_snr{snr:g}_it{iters}_{'et' if et else 'noet'}"
    np.savez_compressed(HERE / f"{tag}.npz", **out)
    print(tag, "FER", float((~conv | words.any(axis=1)).mean()), "mean it", it.mean())


def big_case():
    """z=2500 stand-in, B=2, 3 iterations: hard decisions and a posterior sample."""
    ours = standin_v2(z=2500)
    base = qcldpc.BaseMatrix(ours.n_rows, ours.n_cols, 2500, ours.shifts)
    sched = qcldpc.greedy_schedule(base)
    index = qcldpc.build_compact_index(base, sched)
    n, m = base.n_cols * 2500, base.n_rows * 2500
    llr = channel_llrs(n, 0.161, 0, 0, 2)
    dec = qcldpc.LayeredDecoder(index, sched, qcldpc.DecoderConfig(max_iterations=3, early_termination=False))
    st = dec.new_state(llr)
    syn = np.zeros((2, m), bool)
    for _ in range(3):
        dec._sweep(st, syn)
    sample = np.random.default_rng(7).choice(n, size=20000, replace=False)
    sample.sort()
    np.savez_compressed(
        HERE / "decode_standin_z2500_snr0.161_it3_noet.npz",
        llr_sha=hashlib.sha256(llr.tobytes()).hexdigest(),
        words=np.packbits((st.posterior < 0).astype(np.uint8), axis=1),
        sample_idx=sample, sample_post=st.posterior[:, sample],
    )


def phi_case():
    x = np.concatenate([[0.0, 1e-300, 1e-12, 1e-10, 30.0, 1e6], np.logspace(-10, np.log10(30), 4000)])
    np.savez_compressed(HERE / "phi.npz", x=x, phi=qcldpc.phi(x))


def channel_case():
    rows = []
    for seed, snr, snr_idx, frame, n in [(0, 0.161, 0, 0, 1000), (20240901, 2.5, 12, 5, 800), (3, 1.0, 1, 77, 256)]:
        chan = ChannelConfig(snr=snr, seed=seed)
        llr = init_llr(transmit(np.zeros(n, np.uint8), chan, frame_rng(seed, snr_idx, frame)), chan)
        rows.append((seed, snr, snr_idx, frame, n, hashlib.sha256(llr.tobytes()).hexdigest()))
    with open(HERE / "channel_sha.txt", "w") as fh:
        for r in rows:
            fh.write(" ".join(map(str, r)) + "\n")


def main():
    write_codes()
    phi_case()
    channel_case()
    layer_case("t4x8z3", *ref_code(TEST_BASE_4x8_Z3, 3, merged=False), batch=3, snr=1.0, seed=1)
    layer_case("merge3x3z5", *ref_code(MERGE_EXAMPLE_TOP_PAIR, 5, merged=True), batch=2, snr=1.0, seed=2)
    demo = qcldpc.load_base_matrix(REF_CODES / "demo_4x8_z100.txt")
    dsched = qcldpc.greedy_schedule(demo)
    didx = qcldpc.build_compact_index(demo, dsched)
    layer_case("demo4x8z100", demo, dsched, didx, batch=4, snr=2.5, seed=3)
    ours = standin_v2(z=100)
    sb = qcldpc.BaseMatrix(ours.n_rows, ours.n_cols, 100, ours.shifts)
    ssched = qcldpc.greedy_schedule(sb)
    sidx = qcldpc.build_compact_index(sb, ssched)
    layer_case("standin_z100", sb, ssched, sidx, batch=2, snr=0.161, seed=4)
    for snr in (1.0, 2.5):
        for et in (False, True):
            decode_case("demo4x8z100", demo, dsched, didx, 64, snr, 10, et)
    for snr in (0.161, 0.2):
        for et in (False, True):
            decode_case("standin_z100", sb, ssched, sidx, 16, snr, 50, et, keep_post=(not et and snr == 0.161))
    decode_case("standin_z100", sb, ssched, sidx, 16, 0.161, 10, False, keep_post=True)
    big_case()


if __name__ == "__main__":
    main()

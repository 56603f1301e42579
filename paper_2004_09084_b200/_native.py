"""ctypes binding of ``libqcldpc_b200.so`` (the C ABI in ``include/qcldpc_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a) and is
the only compute path of this package: there is no Python or CPU fallback, and a
missing library is an ImportError the moment a decoder is constructed.  ctypes
releases the GIL for the duration of every call, so one host thread per GPU (or
the reference's ThreadPoolExecutor workers, ``decoder.py:464-472``) run
concurrently.
"""

from __future__ import annotations

import ctypes
import os
import sys
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libqcldpc_b200.so"
# tuning runs (tools/flow_build_variants.sh) may point at an in-tree variant build
if os.environ.get("QCL_LIB_VARIANT"):
    LIB_PATH = LIB_PATH.with_name(f"libqcldpc_b200_{os.environ['QCL_LIB_VARIANT']}.so")

QCL_OK, QCL_EVALUE, QCL_ECUDA, QCL_EUNSUP = 0, -1, -2, -3
PREC = {"fp32": 0, "fp64": 1, "fp32-msg16": 2}  # include/qcldpc_b200.h QCL_PREC_*
DTYPE_F64, DTYPE_F32 = 0, 1


class QclConfig(ctypes.Structure):
    _fields_ = [
        ("max_iterations", ctypes.c_int32),
        ("early_termination", ctypes.c_int32),
        ("llr_clip", ctypes.c_double),
        ("phi_epsilon", ctypes.c_double),
        ("precision", ctypes.c_int32),
    ]


_lib = None
_vp, _i32, _i64, _dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_SIGNATURES = {
    "qcl_abi_version": ([], _i32),
    "qcl_last_error": ([], ctypes.c_char_p),
    "qcl_device_count": ([_vp], ctypes.c_int),
    "qcl_plan_create": ([_i32] * 5 + [_vp] * 6 + [_i32, _vp], ctypes.c_int),
    "qcl_plan_destroy": ([_vp], ctypes.c_int),
    "qcl_plan_info": ([_vp] * 6, ctypes.c_int),
    "qcl_decode": ([_vp, _vp, _vp, _i32, _vp, _i64, _vp, _vp, _vp], ctypes.c_int),
    "qcl_state_create": ([_vp, _i64, _i32, _vp], ctypes.c_int),
    "qcl_state_destroy": ([_vp], ctypes.c_int),
    "qcl_state_set_llr": ([_vp, _vp, _i32], ctypes.c_int),
    "qcl_state_set_llr_synthetic": ([_vp, ctypes.c_uint64, _i64, _i64, _dbl, _i32], ctypes.c_int),
    "qcl_state_set_syndrome": ([_vp, _vp], ctypes.c_int),
    "qcl_state_reset": ([_vp, _dbl], ctypes.c_int),
    "qcl_state_upload": ([_vp, _vp, _vp], ctypes.c_int),
    "qcl_state_download": ([_vp, _vp, _vp], ctypes.c_int),
    "qcl_state_layers": ([_vp, _i32, _i32, _dbl, _dbl], ctypes.c_int),
    "qcl_state_hard_decision": ([_vp, _vp], ctypes.c_int),
    "qcl_state_syndrome_ok": ([_vp, _vp], ctypes.c_int),
    "qcl_state_decode": ([_vp, _vp, _vp], ctypes.c_int),
    "qcl_state_results": ([_vp, _vp, _vp, _vp], ctypes.c_int),
    "qcl_state_truths": ([_vp, _vp], ctypes.c_int),
    "qcl_state_get_llr": ([_vp, _vp], ctypes.c_int),
    "qcl_state_kernel_stats": ([_vp, _vp, _vp, _vp], ctypes.c_int),
    "qcl_state_info": ([_vp, _vp, _vp], ctypes.c_int),
    "qcl_state_set_engine": ([_vp, _i32], ctypes.c_int),
    "qcl_state_frame_errors": ([_vp, _vp], ctypes.c_int),
    "qcl_state_decode_pool": ([_vp, _vp, ctypes.c_uint64, _i64, _i64, _i64, _dbl, _vp, _vp, _vp, _vp], ctypes.c_int),
    "qcl_phi": ([_vp, _i64, _dbl, _dbl, _i32, _i32, _vp], ctypes.c_int),
    "qcl_state_set_syndrome_hint": ([_vp, _vp, _i32], ctypes.c_int),
    "qcl_state_decode_async": ([_vp, _vp], ctypes.c_int),
    "qcl_state_results_async": ([_vp, _vp, _vp, _vp], ctypes.c_int),
    "qcl_state_wait": ([_vp, _vp], ctypes.c_int),
    "qcl_host_alloc": ([_i64, _vp], ctypes.c_int),
    "qcl_host_free": ([_vp], ctypes.c_int),
}
EXPORTED = tuple(_SIGNATURES)


def lib():
    """Load the in-tree library once; fail loudly if it was never built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH.name} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                "this package has no CPU fallback"
            )
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGNATURES.items():
            if os.environ.get("QCL_LIB_VARIANT") and not hasattr(handle, name):
                continue  # an older build under A/B (tools/): symbols it predates are absent
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


def check(rc):
    """Map a C-ABI status to the reference's exception classes."""
    if rc == QCL_OK:
        return
    msg = lib().qcl_last_error().decode("utf-8", "replace")
    if rc == QCL_EVALUE:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def device_count():
    n = ctypes.c_int32(0)
    call("qcl_device_count", ctypes.byref(n))
    return n.value


def make_config(cfg, precision):
    return QclConfig(
        int(cfg.max_iterations),
        int(bool(cfg.early_termination)),
        float(cfg.llr_clip),
        float(cfg.phi_epsilon),
        PREC[precision],
    )


class Plan:
    """Device-resident packed H_compact1 (``qcl_plan``), one per (code, schedule, device)."""

    def __init__(self, index, schedule, device=0):
        from .qc_code import pack_index

        shift, col, off, row = pack_index(index)
        sizes = [len(layer) for layer in schedule.layers]
        starts = np.ascontiguousarray(np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32))
        sched_rows = np.ascontiguousarray(
            np.array([r for layer in schedule.layers for r in layer], dtype=np.int32)
        )
        if len(sched_rows) != len(row):
            raise ValueError("schedule does not match the compact index row order")
        self._keep = (shift, col, off, row, starts, sched_rows)
        self.device = int(device)
        h = ctypes.c_void_p()
        call(
            "qcl_plan_create",
            int(index.z), int(index.n_cols), len(row), len(sizes), int(index.total_edges),
            ptr(shift), ptr(col), ptr(off), ptr(row), ptr(starts), ptr(sched_rows),
            self.device, ctypes.byref(h),
        )
        self.handle = h
        info = [ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()]
        call("qcl_plan_info", h, *(ctypes.byref(x) for x in info))
        self.n, self.m, self.expanded_edges, self.n_layers, self.max_degree = (int(x.value) for x in info)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None and not sys.is_finalizing():  # at exit the process frees it
            _lib.qcl_plan_destroy(h)
            self.handle = None


class State:
    """A device workspace for ``batch`` codewords (``qcl_state``); one host thread at a time."""

    def __init__(self, plan, batch, precision="fp32"):
        self.plan = plan
        self.batch = int(batch)
        self.precision = precision
        h = ctypes.c_void_p()
        call("qcl_state_create", plan.handle, self.batch, PREC[precision], ctypes.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None and not sys.is_finalizing():  # at exit the process frees it
            _lib.qcl_state_destroy(h)
            self.handle = None

    # inputs
    def set_llr(self, llr):
        a = np.ascontiguousarray(llr)
        if a.dtype == np.float32:
            call("qcl_state_set_llr", self.handle, ptr(a), DTYPE_F32)
        else:
            a = np.ascontiguousarray(a, dtype=np.float64)
            call("qcl_state_set_llr", self.handle, ptr(a), DTYPE_F64)

    def set_llr_synthetic(self, seed, snr_idx, first_frame, snr, encode_mode=False):
        call("qcl_state_set_llr_synthetic", self.handle, int(seed) & (2**64 - 1), int(snr_idx),
             int(first_frame), float(snr), int(bool(encode_mode)))

    def set_syndrome(self, syndrome):
        if syndrome is None:
            call("qcl_state_set_syndrome", self.handle, None)
            return
        s = np.ascontiguousarray(syndrome, dtype=np.uint8)
        call("qcl_state_set_syndrome", self.handle, ptr(s))

    # state-level parity API
    def upload(self, posterior, messages=None):
        p = np.ascontiguousarray(posterior, dtype=np.float64)
        m = None if messages is None else np.ascontiguousarray(messages, dtype=np.float64)
        call("qcl_state_upload", self.handle, ptr(p), ptr(m))

    def download(self):
        post = np.empty((self.batch, self.plan.n), np.float64)
        msg = np.empty((self.batch, self.plan.expanded_edges), np.float64)
        call("qcl_state_download", self.handle, ptr(post), ptr(msg))
        return post, msg

    def layers(self, first, count, clip, eps):
        call("qcl_state_layers", self.handle, int(first), int(count), float(clip), float(eps))

    def reset(self, clip):
        call("qcl_state_reset", self.handle, float(clip))

    def hard_decision(self):
        w = np.empty((self.batch, self.plan.n), np.uint8)
        call("qcl_state_hard_decision", self.handle, ptr(w))
        return w

    def syndrome_ok(self):
        ok = np.empty(self.batch, np.uint8)
        call("qcl_state_syndrome_ok", self.handle, ptr(ok))
        return ok.astype(bool)

    # decode
    def decode(self, qcfg):
        ms = ctypes.c_float(0)
        call("qcl_state_decode", self.handle, ctypes.byref(qcfg), ctypes.byref(ms))
        return float(ms.value)

    def results(self, words=True):
        w = np.empty((self.batch, self.plan.n), np.uint8) if words else None
        conv = np.empty(self.batch, np.uint8)
        iters = np.empty(self.batch, np.int64)
        call("qcl_state_results", self.handle, ptr(w), ptr(conv), ptr(iters))
        return w, conv.astype(bool), iters

    def truths(self):
        w = np.empty((self.batch, self.plan.n), np.uint8)
        call("qcl_state_truths", self.handle, ptr(w))
        return w

    def decode_pool(self, qcfg, seed, snr_idx, first_frame, n_frames, snr):
        """Frame pool (qcl_state_decode_pool): per-frame (converged, iterations, frame error), ms."""
        conv = np.empty(n_frames, np.uint8)
        err = np.empty(n_frames, np.uint8)
        iters = np.empty(n_frames, np.int64)
        ms = ctypes.c_float(0)
        call("qcl_state_decode_pool", self.handle, ctypes.byref(qcfg), int(seed) & (2**64 - 1), int(snr_idx),
             int(first_frame), int(n_frames), float(snr), ptr(conv), ptr(iters), ptr(err), ctypes.byref(ms))
        return conv.astype(bool), iters, err.astype(bool), float(ms.value)

    def frame_errors(self):
        """Per frame: decoded word differs from the transmitted one (qcl_state_frame_errors)."""
        out = np.empty(self.batch, np.uint8)
        call("qcl_state_frame_errors", self.handle, ptr(out))
        return out.astype(bool)

    def get_llr(self):
        out = np.empty((self.batch, self.plan.n), np.float64)
        call("qcl_state_get_llr", self.handle, ptr(out))
        return out

    def kernel_stats(self):
        a, b, c = ctypes.c_int64(), ctypes.c_float(), ctypes.c_int64()
        call("qcl_state_kernel_stats", self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        return int(a.value), float(b.value), int(c.value)

    def info(self):
        """(lanes per group, decodes run on the flow engine)"""
        w, f = ctypes.c_int32(), ctypes.c_int32()
        call("qcl_state_info", self.handle, ctypes.byref(w), ctypes.byref(f))
        return int(w.value), bool(f.value)

    def set_engine(self, engine):
        call("qcl_state_set_engine", self.handle, int(engine))

    # asynchronous path
    def set_syndrome_hint(self, syndrome, nonzero=None):
        """nonzero None: the library checks for an all-zero target on its host threads."""
        if syndrome is None or (nonzero is not None and not nonzero):
            call("qcl_state_set_syndrome_hint", self.handle, None, 0)
            return
        call("qcl_state_set_syndrome_hint", self.handle, ptr(syndrome), -1 if nonzero is None else 1)

    def decode_async(self, qcfg):
        call("qcl_state_decode_async", self.handle, ctypes.byref(qcfg))

    def results_async(self, words, conv, iters):
        call("qcl_state_results_async", self.handle, ptr(words), ptr(conv), ptr(iters))

    def wait(self):
        ms = ctypes.c_float(0)
        call("qcl_state_wait", self.handle, ctypes.byref(ms))
        return float(ms.value)


class _PinnedBlock:
    """Owns one qcl_host_alloc block; freed when the last array viewing it is gone."""

    def __init__(self, nbytes):
        p = ctypes.c_void_p()
        call("qcl_host_alloc", max(nbytes, 1), ctypes.byref(p))
        self.ptr = p

    def __del__(self):
        p = getattr(self, "ptr", None)
        if p and p.value and _lib is not None and not sys.is_finalizing():
            _lib.qcl_host_free(p)
            self.ptr = None


class PinnedArray:
    """Page-locked host memory (``qcl_host_alloc``) viewed as a numpy array.

    The memory block is owned by the array's buffer object, so every numpy view of it
    (for example a result yielded by ``decode_stream``) keeps it alive even after this
    wrapper is dropped."""

    def __init__(self, shape, dtype):
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        block = _PinnedBlock(nbytes)
        buf = (ctypes.c_uint8 * max(nbytes, 1)).from_address(block.ptr.value)
        buf._owner = block  # the buffer (the base of every view) keeps the block alive
        self.array = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)


def decode_arrays(plan, qcfg, llr, syndrome):
    """One-shot ``qcl_decode`` on host buffers (the reference-facing hot path)."""
    llr = np.ascontiguousarray(llr)
    if llr.dtype == np.float32:
        dtype = DTYPE_F32
    else:
        llr = np.ascontiguousarray(llr, dtype=np.float64)
        dtype = DTYPE_F64
    batch = llr.shape[0]
    syn = None if syndrome is None else np.ascontiguousarray(syndrome, dtype=np.uint8)
    words = np.empty((batch, plan.n), np.uint8)
    conv = np.empty(batch, np.uint8)
    iters = np.empty(batch, np.int64)
    call("qcl_decode", plan.handle, ctypes.byref(qcfg), ptr(llr), dtype, ptr(syn), batch,
         ptr(words), ptr(conv), ptr(iters))
    return words, conv.astype(bool), iters


def phi_device(x, eps, clip, precision="fp64", device=0):
    a = np.asarray(x, dtype=np.float64)
    flat = np.ascontiguousarray(a.reshape(-1))
    out = np.empty_like(flat)
    call("qcl_phi", ptr(flat), flat.size, float(eps), float(clip), PREC[precision], int(device), ptr(out))
    return out.reshape(a.shape)

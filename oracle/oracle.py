"""ctypes front-end of the CPU oracle (``oracle/layered_ref.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs, never by the
product package.  Every function takes the code as the same four int32 tables
the C-ABI plan takes (see ``paper_2004_09084_b200.qc_code.pack_index``), so a
test can hand the exact same inputs to the oracle and to the CUDA path.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_i32p = ctypes.POINTER(ctypes.c_int32)


class _Code(ctypes.Structure):
    _fields_ = [
        ("z", ctypes.c_int),
        ("n_cols", ctypes.c_int),
        ("n_slots", ctypes.c_int),
        ("n_layers", ctypes.c_int),
        ("n_edges", ctypes.c_int),
        ("edge_shift", _i32p),
        ("edge_col", _i32p),
        ("slot_off", _i32p),
        ("slot_row", _i32p),
        ("layer_start", _i32p),
    ]


def build():
    """Compile liboracle.so with the committed Makefile (gcc, no GPU)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        d, i64, u8p, f64p = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
        L.orc_phi.restype = d
        L.orc_phi.argtypes = [d, d, d]
        L.orc_phi_array.argtypes = [f64p, i64, d, d, f64p]
        L.orc_layer_update.argtypes = [ctypes.c_void_p, ctypes.c_int, f64p, f64p, u8p, i64, d, d]
        L.orc_decode.argtypes = [ctypes.c_void_p, f64p, u8p, i64, ctypes.c_int, ctypes.c_int, d, d,
                                 ctypes.c_int, u8p, u8p, ctypes.c_void_p, f64p]
        L.orc_syndrome.argtypes = [ctypes.c_void_p, u8p, i64, u8p]
        L.orc_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleCode:
    """The code tables in the form the C oracle takes (kept alive with it)."""

    def __init__(self, index, schedule):
        from paper_2004_09084_b200.qc_code import pack_index  # host tables only

        self.shift, self.col, self.off, self.row = pack_index(index)
        sizes = [len(layer) for layer in schedule.layers]
        self.layer_start = np.ascontiguousarray(np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32))
        self.z = int(index.z)
        self.n_cols = int(index.n_cols)
        self.n_slots = len(self.row)
        self.n_layers = len(sizes)
        self.n_edges = int(index.total_edges)
        self.n = self.n_cols * self.z
        self.m = self.n_slots * self.z
        self._c = _Code(
            self.z, self.n_cols, self.n_slots, self.n_layers, self.n_edges,
            *(a.ctypes.data_as(_i32p) for a in (self.shift, self.col, self.off, self.row, self.layer_start)),
        )

    @property
    def ref(self):
        return ctypes.byref(self._c)


def phi(x, eps=1e-10, clip=30.0):
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.empty_like(x)
    lib().orc_phi_array(_ptr(x), x.size, eps, clip, _ptr(out))
    return out


def _syn(code, syndrome, batch):
    if syndrome is None:
        return None
    s = np.ascontiguousarray(np.asarray(syndrome).reshape(batch, code.m).astype(np.uint8))
    return s


def layer_update(code, layer, posterior, messages, syndrome=None, clip=30.0, eps=1e-10):
    """In place on float64 (B, n) / (B, E*z) arrays; ``layer=-1`` runs a full sweep."""
    assert posterior.dtype == np.float64 and posterior.flags.c_contiguous
    assert messages.dtype == np.float64 and messages.flags.c_contiguous
    batch = posterior.shape[0]
    s = _syn(code, syndrome, batch)
    lib().orc_layer_update(code.ref, int(layer), _ptr(posterior), _ptr(messages), _ptr(s), batch, clip, eps)


def decode(code, llr0, syndrome=None, max_iterations=50, early_termination=True, clip=30.0, eps=1e-10,
           threads=0, want_posterior=False):
    """(words u8 (B,n), converged bool (B,), iterations i64 (B,)[, posterior])."""
    llr = np.ascontiguousarray(np.atleast_2d(np.asarray(llr0, dtype=np.float64)))
    batch = llr.shape[0]
    s = _syn(code, syndrome, batch)
    words = np.zeros((batch, code.n), np.uint8)
    conv = np.zeros(batch, np.uint8)
    iters = np.zeros(batch, np.int64)
    post = np.zeros((batch, code.n), np.float64) if want_posterior else None
    lib().orc_decode(code.ref, _ptr(llr), _ptr(s), batch, int(max_iterations), int(bool(early_termination)),
                     clip, eps, int(threads), _ptr(words), _ptr(conv), _ptr(iters), _ptr(post))
    out = (words, conv.astype(bool), iters)
    return out + (post,) if want_posterior else out


def syndrome(code, words):
    w = np.ascontiguousarray(np.atleast_2d(np.asarray(words)).astype(np.uint8))
    out = np.zeros((w.shape[0], code.m), np.uint8)
    lib().orc_syndrome(code.ref, _ptr(w), w.shape[0], _ptr(out))
    return out


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return lib().orc_threads()

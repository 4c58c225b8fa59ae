"""CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product path (``paper_2206_15397_b200``) never does: it fails loudly
when its CUDA library is missing instead of falling back here.

Two interchangeable back ends with one numpy-level API:

* ``port``  -- ``liboracle.so``, the plain-C FP64 restatement in ``rkfac_oracle.c`` (each function cites
  the reference file:line it follows);
* ``ref``   -- ``_ref/librkfac_ref.so``, the UNMODIFIED reference headers compiled where they lie
  (``oracle/Makefile``).  Present wherever it was built (it travels to the GPU box with the snapshot).

The port is pinned to the reference bit-for-bit (``tests/test_oracle.py``) and to the golden fixtures in
``tests/golden/`` that ``tests/golden/make_golden.py`` generated from ``ref``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librkfac_ref.so")  # parity build (-ffp-contract=off, bit-pinned)
REF_STOCK_SO = os.path.join(HERE, "_ref", "librkfac_ref_stock.so")  # timed build: the reference's own flags

STATUS_NAMES = {0: "OK", 1: "DimensionMismatch", 2: "RankDeficient", 3: "NoConvergence",
                4: "DampingNonpositive", 7: "Other"}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {STATUS_NAMES.get(code, code)}")
        self.code = code


def build(targets=("all",)) -> None:
    """Compile the checker (the C restatement, and oracle/_ref when /root/reference is present; "dropin" builds the
    C++ drop-in check against the reference headers and the CUDA library)."""
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class _Lib:
    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix

    def fn(self, name, restype, *argtypes):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        f.argtypes = list(argtypes)
        return f


class Port:
    """numpy API over liboracle.so (the C restatement)."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = _Lib(path, "orc_")
        self._splitmix = L.fn("splitmix64", C.c_uint64, C.c_uint64)
        self._substream = L.fn("substream", C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64)
        self._sample = L.fn("sample_gaussian", C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, C.c_size_t, _dp)
        self._qr = L.fn("qr_thin", C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_int, _dp, _dp)
        self._eig = L.fn("sym_eig", C.c_int, _dp, C.c_size_t, _dp, _dp)
        self._ea = L.fn("ea_update", C.c_int, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double)
        self._srevd = L.fn("srevd", C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64,
                           _u64p, _dp, _dp, _szp)
        self._rsvd = L.fn("rsvd_psd", C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64,
                          _u64p, _dp, _dp, _szp)
        self._apply = L.fn("apply_lowrank_damped_inverse", C.c_int, _dp, _dp, C.c_size_t, C.c_size_t, C.c_double,
                           _dp, C.c_size_t, C.c_size_t, C.c_int, _dp)
        self._apply_eig = L.fn("apply_eig_damped_inverse", C.c_int, _dp, _dp, C.c_size_t, C.c_size_t, C.c_double,
                               _dp, C.c_size_t, C.c_size_t, C.c_int, _dp)
        self._synth = L.fn("synthetic_m", None, C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, C.c_size_t,
                           C.c_double, _dp)

    # rng.hpp
    def splitmix64(self, x: int) -> int:
        return int(self._splitmix(x))

    def substream(self, seed: int, a: int, b: int = 0) -> int:
        return int(self._substream(seed, a, b))

    def sample_gaussian(self, seed: int, counter: int, m: int, n: int):
        out = np.empty((m, n), np.float64)
        ctr = self._sample(seed, counter, m, n, _ptr(out))
        return out, int(ctr)

    # qr.hpp / eig.hpp
    def qr_thin(self, x, strict: bool = False):
        x = _f64(x)
        m, n = x.shape
        q = np.empty((m, n)); r = np.empty((n, n))
        st = self._qr(_ptr(x), m, n, int(strict), _ptr(q), _ptr(r))
        if st:
            raise OracleError(st, "qr_thin")
        return q, r

    def sym_eig(self, s):
        s = _f64(s)
        n = s.shape[0]
        p = np.empty((n, n)); d = np.empty(n)
        st = self._eig(_ptr(s), n, _ptr(p), _ptr(d))
        if st:
            raise OracleError(st, "sym_eig")
        return p, d

    # kfactor.hpp / rnla.hpp
    def ea_update(self, mbar, m, rho: float) -> np.ndarray:
        out = _f64(mbar).copy()
        m = _f64(m)
        st = self._ea(_ptr(out), out.shape[0], _ptr(m), m.shape[0], m.shape[1], rho)
        if st:
            raise OracleError(st, "ea_update")
        return out

    def _decomp(self, f, name, x, r, p, q, seed, counter):
        x = _f64(x)
        d = x.shape[0]
        u = np.empty((d, max(1, min(r, d)))); dv = np.empty(max(1, min(r, d)))
        ctr = C.c_uint64(counter); rout = C.c_size_t(0)
        st = f(_ptr(x), d, r, p, q, seed, C.byref(ctr), _ptr(u), _ptr(dv), C.byref(rout))
        if st:
            raise OracleError(st, name)
        rr = rout.value
        return u[:, :rr].copy(), dv[:rr].copy(), int(ctr.value)

    def srevd(self, x, r, p, q, seed, counter=0):
        return self._decomp(self._srevd, "srevd", x, r, p, q, seed, counter)

    def rsvd_psd(self, x, r, p, q, seed, counter=0):
        return self._decomp(self._rsvd, "rsvd_psd", x, r, p, q, seed, counter)

    def apply_lowrank_damped_inverse(self, u, dv, lam: float, v, side: str):
        u = _f64(u); dv = _f64(dv); v = _f64(v)
        out = np.empty_like(v)
        st = self._apply(_ptr(u), _ptr(dv), u.shape[0], u.shape[1], lam, _ptr(v), v.shape[0], v.shape[1],
                         0 if side == "left" else 1, _ptr(out))
        if st:
            raise OracleError(st, "apply_lowrank_damped_inverse")
        return out

    def apply_eig_damped_inverse(self, u, dv, lam: float, v, side: str):
        u = _f64(u); dv = _f64(dv); v = _f64(v)
        out = np.empty_like(v)
        st = self._apply_eig(_ptr(u), _ptr(dv), u.shape[0], u.shape[1], lam, _ptr(v), v.shape[0], v.shape[1],
                             0 if side == "left" else 1, _ptr(out))
        if st:
            raise OracleError(st, "apply_eig_damped_inverse")
        return out

    def precondition(self, ua, da, ug, dg, lam: float, j):
        """optimizer.hpp:159-162: LEFT_G(RIGHT_A(J))."""
        mid = self.apply_lowrank_damped_inverse(ua, da, lam, j, "right")
        return self.apply_lowrank_damped_inverse(ug, dg, lam, mid, "left")

    def synthetic_m(self, root: int, step: int, f: int, n: int, d: int, e: float) -> np.ndarray:
        m = np.empty((d, n))
        self._synth(root, step, f, n, d, e, _ptr(m))
        return m


class Ref(Port):
    """The same numpy API over the reference's own code (oracle/_ref/librkfac_ref.so)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):  # noqa: D107 -- different symbol set, explicit bindings
        L = _Lib(path, "ref_")
        self._port = Port()
        self._substream_r = L.fn("substream", C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64)
        self._sample_r = L.fn("sample_gaussian", C.c_int, C.c_uint64, C.c_uint64, C.c_size_t, C.c_size_t, _dp,
                              _u64p)
        self._qr = L.fn("qr_thin", C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_int, _dp, _dp)
        self._eig = L.fn("sym_eig", C.c_int, _dp, C.c_size_t, _dp, _dp)
        self._ea = L.fn("ea_update", C.c_int, _dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_double)
        self._dec = L.fn("decompose", C.c_int, C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                         C.c_uint64, _u64p, _dp, _dp, _szp)
        self._apply = L.fn("apply_lowrank", C.c_int, _dp, _dp, C.c_size_t, C.c_size_t, C.c_double, _dp,
                           C.c_size_t, C.c_size_t, C.c_int, _dp)
        self._rsvd = L.fn("rsvd", C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                          C.c_uint64, _u64p, _dp, _dp, _dp, _szp)
        self._step = L.fn("step_threaded", C.c_int, C.c_int, C.c_int, C.c_size_t, _szp, _szp,
                          C.POINTER(_dp), C.POINTER(_dp), _szp, C.c_double, C.c_size_t, C.c_size_t, C.c_size_t,
                          C.c_uint64, C.c_uint64, C.c_double, C.POINTER(_dp), C.POINTER(_dp), _dp,
                          C.POINTER(_dp), C.POINTER(_dp))

    def splitmix64(self, x):
        return self._port.splitmix64(x)

    def substream(self, seed, a, b=0):
        return int(self._substream_r(seed, a, b))

    def sample_gaussian(self, seed, counter, m, n):
        out = np.empty((m, n)); ctr = C.c_uint64(0)
        st = self._sample_r(seed, counter, m, n, _ptr(out), C.byref(ctr))
        if st:
            raise OracleError(st, "sample_gaussian")
        return out, int(ctr.value)

    def _decomp_m(self, method, name, x, r, p, q, seed, counter):
        x = _f64(x)
        d = x.shape[0]
        u = np.empty((d, max(1, min(r, d)))); dv = np.empty(max(1, min(r, d)))
        ctr = C.c_uint64(counter); rout = C.c_size_t(0)
        st = self._dec(method, _ptr(x), d, r, p, q, seed, C.byref(ctr), _ptr(u), _ptr(dv), C.byref(rout))
        if st:
            raise OracleError(st, name)
        rr = rout.value
        return np.ascontiguousarray(u.reshape(-1)[: d * rr].reshape(d, rr)), dv[:rr].copy(), int(ctr.value)

    def srevd(self, x, r, p, q, seed, counter=0):
        return self._decomp_m(0, "srevd", x, r, p, q, seed, counter)

    def rsvd_psd(self, x, r, p, q, seed, counter=0):
        return self._decomp_m(1, "rsvd_psd", x, r, p, q, seed, counter)

    def rsvd(self, x, r, p, q, seed, counter=0):
        """rnla.hpp:62-77 on a general matrix: (u, s, v, counter)."""
        x = _f64(x)
        rows, cols = x.shape
        k = max(1, min(r, rows, cols))
        u = np.empty((rows, k)); s = np.empty(k); v = np.empty((cols, k))
        ctr = C.c_uint64(counter); rout = C.c_size_t(0)
        st = self._rsvd(_ptr(x), rows, cols, r, p, q, seed, C.byref(ctr), _ptr(u), _ptr(s), _ptr(v), C.byref(rout))
        if st:
            raise OracleError(st, "rsvd")
        rr = rout.value
        return (np.ascontiguousarray(u.reshape(-1)[: rows * rr].reshape(rows, rr)), s[:rr].copy(),
                np.ascontiguousarray(v.reshape(-1)[: cols * rr].reshape(cols, rr)), int(ctr.value))

    def apply_eig_damped_inverse(self, *a, **k):
        return self._port.apply_eig_damped_inverse(*a, **k)

    def synthetic_m(self, *a, **k):
        return self._port.synthetic_m(*a, **k)

    def step_threaded(self, method: str, threads: int, dims_a, dims_g, factors, ms, ns, rho, r, p, q,
                      rng_root, step, lam, grads, outs, us=None, dvs=None):
        """The reference's EA -> decompositions -> preconditioning over layers, one factor per thread.  Optional
        us / dvs (per factor, d x min(r, d) and min(r, d) FP64 arrays) receive the decompositions."""
        nl = len(dims_a)
        A = (C.c_size_t * nl)(*dims_a)
        G = (C.c_size_t * nl)(*dims_g)
        fp = (_dp * (2 * nl))(*[_ptr(f) for f in factors])
        mp = (_dp * (2 * nl))(*[_ptr(m) for m in ms]) if ms is not None else None
        nn = (C.c_size_t * (2 * nl))(*ns) if ns is not None else None
        gp = (_dp * nl)(*[_ptr(g) for g in grads]) if grads is not None else None
        op = (_dp * nl)(*[_ptr(o) for o in outs]) if outs is not None else None
        up = (_dp * (2 * nl))(*[_ptr(u) for u in us]) if us is not None else None
        dp = (_dp * (2 * nl))(*[_ptr(x) for x in dvs]) if dvs is not None else None
        ph = np.zeros(3)
        st = self._step(0 if method == "srevd" else 1, threads, nl, A, G, fp, mp, nn, rho, r, p, q, rng_root,
                        step, lam, gp, op, _ptr(ph), up, dp)
        if st:
            raise OracleError(st, "step_threaded")
        return ph


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def best() -> Port:
    """The reference build when present, else the restatement."""
    return ref() if ref_available() else port()


_ref_stock = None


def ref_stock() -> Ref:
    """The reference compiled with its own flags (proj/CMakeLists.txt:9) -- the CPU baseline that bench.py times."""
    global _ref_stock
    if _ref_stock is None:
        _ref_stock = Ref(REF_STOCK_SO)
    return _ref_stock


def ref_stock_available() -> bool:
    return os.path.exists(REF_STOCK_SO)


def parallel_map(fn, items, threads: int):
    """ctypes releases the GIL, so oracle calls on distinct data run concurrently."""
    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        return list(ex.map(fn, items))

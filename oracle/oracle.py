"""TEST INFRASTRUCTURE ONLY — numpy-facing ctypes wrappers over

* ``LcOracle``  : our fp64 C restatement (oracle/lc_oracle.c -> build/liblcoracle.so)
* ``RefOracle`` : the unmodified reference compiled in place
                  (oracle/ref_capi.cpp + /root/reference/proj/src -> _ref/liblongconv_ref.so)

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
(paper_2302_06646_b200) never does.  Both classes expose the same method
names so parity tests can run against either.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LC_LIB = HERE / "build" / "liblcoracle.so"
REF_LIB = HERE / "_ref" / "liblongconv_ref.so"

_sz = C.c_size_t
_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _cplx_in(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a.view(np.float64)


def _cplx_out(n: int) -> np.ndarray:
    return np.zeros(2 * n, dtype=np.float64)


def build_oracles(with_ref: bool | None = None) -> None:
    """Compile the oracle libraries (make -C oracle).  The reference library
    is only (re)built when /root/reference is present."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if with_ref is None:
        with_ref = Path("/root/reference/proj/src").is_dir()
    if with_ref:
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


class _Base:
    prefix = ""
    LIB: Path

    def __init__(self):
        if not self.LIB.exists():
            raise FileNotFoundError(f"{self.LIB} missing: run `make -C oracle`")
        self.lib = C.CDLL(str(self.LIB))

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _call(self, name, *args):
        rc = self._f(name)(*args)
        if rc != 0:
            raise ValueError(f"{self.prefix}{name} failed with code {rc}: {self._err()}")

    def _err(self):
        return ""

    # -- rng / init ------------------------------------------------------
    def normal_draws(self, seed, stream, count):
        out = np.zeros(count)
        self._call("normal_draws", _u64(seed), _u64(stream), _sz(count), _ptr(out))
        return out

    def uniform_draws(self, seed, stream, count):
        out = np.zeros(count)
        self._call("uniform_draws", _u64(seed), _u64(stream), _sz(count), _ptr(out))
        return out

    def signal_batch(self, seed, B, H, N):
        """u[b,h,:] = standard_normal_draws(SeededRng(seed).child(b*H+h), N)."""
        if self.prefix != "lco_":
            out = np.stack([self.normal_draws(seed, c, N) for c in range(B * H)])
            return out.reshape(B, H, N)
        out = np.zeros((B, H, N))
        self._call("signal_batch", _u64(seed), _sz(B), _sz(H), _sz(N), _ptr(out))
        return out

    def init_kernels(self, kind, H, N, seed):
        """kind: 0 random, 1 geometric (regularize.cpp:73-91) -> (K[H,N], D[H])."""
        K = np.zeros((H, N))
        D = np.zeros(H)
        self._call("init_kernels", C.c_int(kind), _sz(H), _sz(N), _u64(seed), _ptr(K), _ptr(D))
        return K, D

    # -- regularizers ----------------------------------------------------
    def squash(self, k, lam):
        k = _f64(k)
        out = np.zeros_like(k)
        self._call("squash", _ptr(k), _sz(k.size), C.c_double(lam), _ptr(out))
        return out

    def smooth(self, k, p):
        k = _f64(k)
        out = np.zeros_like(k)
        self._call("smooth", _ptr(k), _sz(k.size), _sz(p), _ptr(out))
        return out

    def smooth_frequency(self, k, p):
        k = _f64(k)
        out = np.zeros_like(k)
        self._call("smooth_frequency", _ptr(k), _sz(k.size), _sz(p), _ptr(out))
        return out

    def regularize_bank(self, K, lam, p, rate=0.0, domain=0, seed=0, training=False):
        K = _f64(K)
        H, N = K.shape
        out = np.zeros_like(K)
        self._call("regularize_bank", *self._bank_args(K, H, N), C.c_double(lam), _sz(p),
                   C.c_double(rate), C.c_int(domain), _u64(seed), C.c_int(int(training)),
                   _ptr(out))
        return out

    def _bank_args(self, K, H, N):
        return (_ptr(K), _sz(H), _sz(N))

    def regularizer_backward(self, K, lam, p, dKbar, rate=0.0, seed=0, training=False):
        K = _f64(K)
        dKbar = _f64(dKbar)
        H, N = K.shape
        out = np.zeros_like(K)
        self._call("regularizer_backward", _ptr(K), _sz(H), _sz(N), C.c_double(lam), _sz(p),
                   C.c_double(rate), _u64(seed), C.c_int(int(training)), _ptr(dKbar),
                   _ptr(out))
        return out

    # -- transforms ------------------------------------------------------
    def plan_factors(self, n, r=16):
        f = (C.c_size_t * 64)()
        cnt = C.c_size_t(0)
        self._call("plan_factors", _sz(n), _sz(r), f, C.byref(cnt))
        return [int(f[i]) for i in range(cnt.value)]

    def apply_plan(self, x, r=16, inverse=False):
        xin = _cplx_in(x)
        n = xin.size // 2
        out = _cplx_out(n)
        self._call("apply_plan", _sz(n), _sz(r), _ptr(xin), C.c_int(int(inverse)), _ptr(out))
        return out.view(np.complex128)

    def dft_naive(self, x, inverse=False):
        xin = _cplx_in(x)
        n = xin.size // 2
        out = _cplx_out(n)
        self._call("dft_naive", _ptr(xin), _sz(n), C.c_int(int(inverse)), _ptr(out))
        return out.view(np.complex128)

    def conv_butterfly(self, u, k, causal=True):
        uin, kin = _cplx_in(u), _cplx_in(k)
        n = uin.size // 2
        out = _cplx_out(n)
        self._call("conv_butterfly", _ptr(uin), _ptr(kin), _sz(n), C.c_int(int(causal)),
                   _ptr(out))
        return out.view(np.complex128)

    def conv_naive_real(self, u, k, causal=True):
        u, k = _f64(u), _f64(k)
        out = np.zeros_like(u)
        self._call("conv_naive_real", _ptr(u), _ptr(k), _sz(u.size), C.c_int(int(causal)),
                   _ptr(out))
        return out

    def conv_three_pass(self, u, k, l, m):
        uin, kin = _cplx_in(u), _cplx_in(k)
        n = uin.size // 2
        out = _cplx_out(n)
        self._call_three_pass(uin, kin, n, l, m, out)
        return out.view(np.complex128)

    def _call_three_pass(self, uin, kin, n, l, m, out):
        self._call("conv_three_pass", _ptr(uin), _ptr(kin), _sz(n), _sz(l), _sz(m), _ptr(out))

    def three_pass_dk(self, k, l, m):
        kin = _cplx_in(k)
        n = kin.size // 2
        out = _cplx_out(n)
        self._call("three_pass_dk", _ptr(kin), _sz(n), _sz(l), _sz(m), _ptr(out))
        return out.view(np.complex128)

    def conv_real_packed(self, u, k, causal=True):
        u, k = _f64(u), _f64(k)
        out = np.zeros_like(u)
        self._call("conv_real_packed", _ptr(u), _ptr(k), _sz(u.size), C.c_int(int(causal)),
                   _ptr(out))
        return out

    # -- learned butterfly -----------------------------------------------
    def learned_param_count(self, n, r=16):
        c = C.c_size_t(0)
        self._call("learned_param_count", _sz(n), _sz(r), C.byref(c))
        return c.value

    def learned_init(self, n, r=16):
        out = _cplx_out(self.learned_param_count(n, r))
        self._call("learned_init", _sz(n), _sz(r), _ptr(out))
        return out.view(np.complex128)

    def learned_forward(self, blocks, x, r=16):
        b, xin = _cplx_in(blocks), _cplx_in(x)
        n = xin.size // 2
        out = _cplx_out(n)
        self._call("learned_forward", _sz(n), _sz(r), _ptr(b), _ptr(xin), _ptr(out))
        return out.view(np.complex128)

    def learned_gradients(self, blocks, x, g, r=16):
        b, xin, gin = _cplx_in(blocks), _cplx_in(x), _cplx_in(g)
        n = xin.size // 2
        db = np.zeros_like(b)
        dx = _cplx_out(n)
        self._call("learned_gradients", _sz(n), _sz(r), _ptr(b), _ptr(xin), _ptr(gin), _ptr(db),
                   _ptr(dx))
        return db.view(np.complex128), dx.view(np.complex128)


class LcOracle(_Base):
    """Our fp64 C restatement (lc_oracle.c)."""

    prefix = "lco_"
    LIB = LC_LIB

    def long_conv_forward(self, u, Kbar, D, causal=True):
        u, Kbar, D = _f64(u), _f64(Kbar), _f64(D)
        B, H, N = u.shape
        y = np.zeros_like(u)
        self._call("long_conv_forward", _ptr(u), _sz(B), _sz(H), _sz(N), _ptr(Kbar), _ptr(D),
                   C.c_int(int(causal)), _ptr(y))
        return y

    def regularized_long_conv(self, u, K, D, lam=0.0, p=0, rate=0.0, domain=0, seed=0,
                              causal=True, training=False):
        u, K, D = _f64(u), _f64(K), _f64(D)
        B, H, N = u.shape
        y = np.zeros_like(u)
        self._call("regularized_long_conv", _ptr(u), _sz(B), _sz(H), _sz(N), _ptr(K), _ptr(D),
                   C.c_double(lam), _sz(p), C.c_double(rate), C.c_int(domain), _u64(seed),
                   C.c_int(int(causal)), C.c_int(int(training)), _ptr(y))
        return y

    def long_conv_backward(self, u, dy, Kbar, D, causal=True):
        """-> (du[B,H,N], dKbar[H,N], dD[H]) w.r.t. the REGULARIZED kernel."""
        u, dy, Kbar, D = _f64(u), _f64(dy), _f64(Kbar), _f64(D)
        B, H, N = u.shape
        du = np.zeros_like(u)
        dK = np.zeros((H, N))
        dD = np.zeros(H)
        self._call("long_conv_backward", _ptr(u), _ptr(dy), _sz(B), _sz(H), _sz(N), _ptr(Kbar),
                   _ptr(D), C.c_int(int(causal)), _ptr(du), _ptr(dK), _ptr(dD))
        return du, dK, dD


class RefOracle(_Base):
    """The unmodified reference library (via oracle/ref_capi.cpp)."""

    prefix = "ref_"
    LIB = REF_LIB

    def __init__(self, threads: int | None = None):
        super().__init__()
        self.lib.ref_last_error.restype = C.c_char_p
        self.threads = threads or os.cpu_count() or 1

    def _err(self):
        return self.lib.ref_last_error().decode()

    def _bank_args(self, K, H, N):
        D = np.zeros(H)
        self._keep = D
        return (_ptr(K), _ptr(D), _sz(H), _sz(N))

    def _call_three_pass(self, uin, kin, n, l, m, out):
        sweeps = C.c_int(0)
        self._call("conv_three_pass", _ptr(uin), _ptr(kin), _sz(n), _sz(l), _sz(m), _ptr(out),
                   C.byref(sweeps))
        self.last_sweeps = sweeps.value

    def regularized_long_conv(self, u, K, D, lam=0.0, p=0, rate=0.0, domain=0, seed=0,
                              causal=True, training=False, engine=1, threads=None):
        """engine: 0 naive, 1 butterfly, 2 three-pass (regularize.hpp:17)."""
        u, K, D = _f64(u), _f64(K), _f64(D)
        B, H, N = u.shape
        y = np.zeros_like(u)
        self._call("regularized_long_conv", _ptr(u), _sz(B), _sz(H), _sz(N), _ptr(K), _ptr(D),
                   C.c_double(lam), _sz(p), C.c_double(rate), C.c_int(domain), _u64(seed),
                   C.c_int(engine), C.c_int(int(causal)), C.c_int(int(training)),
                   C.c_int(threads or self.threads), _ptr(y))
        return y

    def long_conv_forward(self, u, Kbar, D, causal=True, engine=1, threads=None):
        return self.regularized_long_conv(u, Kbar, D, causal=causal, engine=engine,
                                          threads=threads)

    def long_conv_backward(self, u, dy, Kbar, D, causal=True, threads=None):
        """Composed from reference conv_butterfly (causal only)."""
        assert causal, "the composed reference backward is causal-only"
        u, dy, Kbar, D = _f64(u), _f64(dy), _f64(Kbar), _f64(D)
        B, H, N = u.shape
        du = np.zeros_like(u)
        dK = np.zeros((H, N))
        dD = np.zeros(H)
        self._call("long_conv_backward", _ptr(u), _ptr(dy), _sz(B), _sz(H), _sz(N), _ptr(Kbar),
                   _ptr(D), C.c_int(threads or self.threads), _ptr(du), _ptr(dK), _ptr(dD))
        return du, dK, dD


def ref_available() -> bool:
    return REF_LIB.exists()


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.complex128 if np.iscomplexobj(a) else np.float64)
    b = np.asarray(b, dtype=a.dtype)
    den = np.linalg.norm(b.ravel())
    num = np.linalg.norm((a - b).ravel())
    return float(num / den) if den > 0 else float(num)

"""Host-side mirror of the reference learned butterfly (K5) on the C ABI.

* :class:`LearnedButterflyPlan` <- ``LearnedButterfly`` (butterfly.hpp:88-94):
  the stage scaffolding of ``build_plan(n, r)`` with one trainable f x f
  complex block per stage, here per head.
* :meth:`LearnedButterflyPlan.forward`   <- ``learned_forward``  (butterfly.hpp:96)
* :meth:`LearnedButterflyPlan.gradients` <- ``learned_gradients`` (butterfly.hpp:104-106)
* :func:`learned_butterfly`            — differentiable torch op

Rows are [B, H, n] complex: ``torch.complex64`` for the fp32 mode, or
``[B, H, n, 2]`` bf16/fp16 (interleaved re/im) for the 16-bit modes.  Blocks
are ``[H, P]`` complex64 (P = sum_s f_s^2, stages concatenated).
Gradients follow the reference (and PyTorch) convention dJ/dRe + i dJ/dIm
for J = Re <upstream, y>.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import DimensionError, check
from .longconv import _ptr, _stream

_DT = {torch.complex64: _lib.FB_F32, torch.float32: _lib.FB_F32, torch.bfloat16: _lib.FB_BF16,
       torch.float16: _lib.FB_F16}


class LearnedButterflyPlan:
    def __init__(self, n: int, r: int = 16, H: int = 1, dtype: torch.dtype = torch.complex64,
                 device=None):
        if dtype not in _DT:
            raise TypeError(f"unsupported dtype {dtype}")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.n, self.r, self.H, self.dtype, self.device = int(n), int(r), int(H), dtype, dev
        h = C.c_void_p()
        check(_lib.lib().fb_learned_plan_create(C.byref(h), self.n, self.r, self.H, _DT[dtype],
                                                dev.index or 0))
        self._h = h
        f = (C.c_int64 * 32)()
        cnt, pc = C.c_int64(), C.c_int64()
        check(_lib.lib().fb_learned_plan_factors(h, f, C.byref(cnt), C.byref(pc)))
        self.factors = [int(f[i]) for i in range(cnt.value)]
        self.param_count = int(pc.value)
        eng = C.c_int()
        check(_lib.lib().fb_learned_plan_engine(h, C.byref(eng)))
        # kernel family: generic stage walk, CUDA-core fast path, or tcgen05
        self.engine = ("generic", "cuda-core", "tcgen05")[eng.value]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().fb_learned_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def dft_blocks(self) -> torch.Tensor:
        """Blocks of LearnedButterfly::from_plan (butterfly.cpp:221-227): the
        f-point DFT matrices exp(-2 pi i ((p q) mod f) / f), for every head."""
        parts = []
        for f in self.factors:
            pq = (np.arange(f)[:, None] * np.arange(f)[None, :]) % f
            parts.append(np.exp(-2j * np.pi * pq / f).ravel())
        one = torch.tensor(np.concatenate(parts), dtype=torch.complex64)
        return one.unsqueeze(0).repeat(self.H, 1).to(self.device)

    def _rows(self, x: torch.Tensor, name: str) -> int:
        want_c = self.dtype in (torch.complex64, torch.float32)
        shape_ok = (x.dim() == 3 and x.shape[1:] == (self.H, self.n)) if want_c else \
            (x.dim() == 4 and x.shape[1:] == (self.H, self.n, 2))
        if not shape_ok:
            raise DimensionError(_lib.FB_ERR_DIM, f"{name}: bad shape {list(x.shape)}")
        if want_c and x.dtype != torch.complex64:
            raise TypeError(f"{name}: expected complex64")
        if not want_c and x.dtype != self.dtype:
            raise TypeError(f"{name}: expected {self.dtype}")
        if not x.is_contiguous() or x.device != self.device:
            raise TypeError(f"{name}: expected contiguous on {self.device}")
        return x.shape[0]

    def _blocks(self, blocks: torch.Tensor) -> torch.Tensor:
        if blocks.shape != (self.H, self.param_count):
            raise DimensionError(_lib.FB_ERR_DIM, "learned: block count != stage count")
        return blocks.to(self.device, torch.complex64).contiguous()

    def forward(self, blocks: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        B = self._rows(x, "x")
        blocks = self._blocks(blocks)
        y = torch.empty_like(x)
        check(_lib.lib().fb_learned_fwd(self._h, _ptr(blocks), _ptr(x), _ptr(y), B, C.c_void_p(0),
                                        _stream(self.device)))
        return y

    def gradients(self, blocks: torch.Tensor, x: torch.Tensor, upstream: torch.Tensor):
        """-> (block_grads [H, P] summed over b, input_grad like x)."""
        B = self._rows(x, "x")
        if self._rows(upstream, "upstream") != B:
            raise DimensionError(_lib.FB_ERR_DIM, "learned_gradients: shape mismatch")
        blocks = self._blocks(blocks)
        dx = torch.empty_like(x)
        db = torch.empty_like(blocks)
        nbytes = _lib.lib().fb_learned_workspace_size(self._h, B)
        ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.device)
        check(_lib.lib().fb_learned_bwd(self._h, _ptr(blocks), _ptr(x), _ptr(upstream), _ptr(dx),
                                        _ptr(db), B, _ptr(ws), _stream(self.device)))
        return db, dx


_PLANS: dict = {}


def _plan(n, r, H, dtype, device):
    key = (n, r, H, dtype, str(device))
    if key not in _PLANS:
        _PLANS[key] = LearnedButterflyPlan(n, r, H, dtype, device)
    return _PLANS[key]


class _LearnedFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, blocks, r):
        H, n = x.shape[1], x.shape[2]
        plan = _plan(n, r, H, x.dtype, x.device)
        ctx.save_for_backward(x, blocks)
        ctx.plan = plan
        return plan.forward(blocks, x.contiguous())

    @staticmethod
    def backward(ctx, g):
        x, blocks = ctx.saved_tensors
        db, dx = ctx.plan.gradients(blocks, x, g.contiguous())
        return dx, db.to(blocks.dtype), None


def learned_butterfly(x: torch.Tensor, blocks: torch.Tensor, r: int = 16) -> torch.Tensor:
    """y[b, h] = LearnedButterfly_h(x[b, h]) with trainable blocks [H, P]."""
    return _LearnedFn.apply(x, blocks, r)


class LearnedLongConvPlan:
    """The learned-butterfly long convolution: FlashButterfly
    with the Butterfly matrices of its transform learned (fb_lconv_* in
    libflashbutterfly.so).  Per head h:
        y = Re IL(Wi[h], L(Wf[h], pad u) * L(Wf[h], pad Kbar[h]))[:N] + D[h] u
    with L = learned_forward over build_plan(n, r) and IL(W, z) =
    conj(L(W, conj z)) / n; n = 2N causal, N circular.  fp32 signals
    [B, H, N]; blocks Wf, Wi [H, P] complex64.  dft_blocks() initialises both
    to the DFT, where the operator equals regularized_long_conv."""

    def __init__(self, N: int, H: int, r: int = 16, mode=1, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.N, self.H, self.r, self.mode, self.device = int(N), int(H), int(r), int(mode), dev
        h = C.c_void_p()
        check(_lib.lib().fb_lconv_plan_create(C.byref(h), self.N, self.H, self.r, self.mode, dev.index or 0))
        self._h = h
        n, pc = C.c_int64(), C.c_int64()
        check(_lib.lib().fb_lconv_plan_dims(h, C.byref(n), C.byref(pc)))
        self.n, self.param_count = int(n.value), int(pc.value)
        self._lb = LearnedButterflyPlan(self.n, self.r, self.H, torch.complex64, dev)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().fb_lconv_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def dft_blocks(self) -> torch.Tensor:
        return self._lb.dft_blocks()

    def _ws(self, B):
        return torch.empty(max(int(_lib.lib().fb_lconv_workspace_size(self._h, B)), 1), dtype=torch.uint8,
                           device=self.device)

    def _check(self, u):
        if u.dim() != 3 or u.shape[1:] != (self.H, self.N):
            raise DimensionError(_lib.FB_ERR_DIM, f"learned conv: expected [B, {self.H}, {self.N}]")
        return u.shape[0]

    @staticmethod
    def _f(t, dt=torch.float32):
        return t.detach().to(dtype=dt).contiguous()

    def forward(self, u, kbar, D, Wf, Wi):
        B = self._check(u)
        u, kbar, D = self._f(u), self._f(kbar), self._f(D)
        Wf, Wi = self._f(Wf, torch.complex64), self._f(Wi, torch.complex64)
        y = torch.empty_like(u)
        check(_lib.lib().fb_lconv_fwd(self._h, _ptr(u), _ptr(kbar), _ptr(D), _ptr(Wf), _ptr(Wi), _ptr(y), B,
                                      _ptr(self._ws(B)), _stream(self.device)))
        return y

    def backward(self, dy, u, kbar, D, Wf, Wi):
        """-> (du, dKbar, dD, dWf, dWi)."""
        B = self._check(u)
        dy, u, kbar, D = self._f(dy), self._f(u), self._f(kbar), self._f(D)
        Wf, Wi = self._f(Wf, torch.complex64), self._f(Wi, torch.complex64)
        du, dk, dD = torch.empty_like(u), torch.empty_like(kbar), torch.empty_like(D)
        dWf, dWi = torch.empty_like(Wf), torch.empty_like(Wi)
        check(_lib.lib().fb_lconv_bwd(self._h, _ptr(dy), _ptr(u), _ptr(kbar), _ptr(D), _ptr(Wf), _ptr(Wi),
                                      _ptr(du), _ptr(dk), _ptr(dD), _ptr(dWf), _ptr(dWi), B, _ptr(self._ws(B)),
                                      _stream(self.device)))
        return du, dk, dD, dWf, dWi


class _LearnedConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, u, kbar, D, Wf, Wi, plan):
        ctx.save_for_backward(u, kbar, D, Wf, Wi)
        ctx.plan = plan
        return plan.forward(u, kbar, D, Wf, Wi)

    @staticmethod
    def backward(ctx, dy):
        u, kbar, D, Wf, Wi = ctx.saved_tensors
        du, dk, dD, dWf, dWi = ctx.plan.backward(dy, u, kbar, D, Wf, Wi)
        return du, dk, dD, dWf.to(Wf.dtype), dWi.to(Wi.dtype), None


def learned_long_conv(u, kbar, D, Wf, Wi, r: int = 16, mode: int = 1):
    """Differentiable learned-butterfly long convolution (see LearnedLongConvPlan)."""
    key = ("lconv", u.shape[2], u.shape[1], r, mode, str(u.device))
    if key not in _PLANS:
        _PLANS[key] = LearnedLongConvPlan(u.shape[2], u.shape[1], r, mode, u.device)
    return _LearnedConvFn.apply(u, kbar, D, Wf, Wi, _PLANS[key])

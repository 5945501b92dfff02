"""Host-side mirror of the reference ``longconv`` layer API on top of the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/longconv/regularize.hpp and butterfly.hpp:

* :class:`RegularizationConfig`  <- ``RegularizationConfig`` (regularize.hpp:19-25)
* :class:`Engine`, :class:`ConvMode`, :class:`SmoothDomain` <- the reference enums
* :func:`regularized_long_conv`  <- ``regularized_long_conv`` (regularize.hpp:67-70)
* :func:`regularized_long_conv_backward` — the backward the reference lacks
* :func:`long_conv`              — differentiable (torch.autograd) form
* :class:`LongConvPlan`          — explicit plan handle (``fb_plan``)

Tensors are torch CUDA tensors laid out like ``SignalBatch`` [B, H, N] and
``KernelBank`` ([H, N] kernels + [H] skip gains).  All compute happens in
libflashbutterfly.so on the current CUDA stream; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import DimensionError, FBError, PlanError, check  # noqa: F401 (re-export)


class Engine(enum.IntEnum):
    """Execution path (regularize.hpp:17).  kNaive stays in the CPU oracle;
    AUTO picks single-pass when the transform fits in shared memory."""

    AUTO = _lib.FB_ENGINE_AUTO
    BUTTERFLY = _lib.FB_ENGINE_SINGLE  # single-pass fused kernel
    THREE_PASS = _lib.FB_ENGINE_THREE
    BUTTERFLY_SIMT = _lib.FB_ENGINE_SINGLE_SIMT  # single-pass on CUDA cores (fp32 FFT)


class ConvMode(enum.IntEnum):  # butterfly.hpp:69
    CIRCULAR = _lib.FB_MODE_CIRCULAR
    CAUSAL = _lib.FB_MODE_CAUSAL


class SmoothDomain(enum.IntEnum):  # regularize.hpp:16
    TIME = _lib.FB_SMOOTH_TIME
    FREQUENCY = _lib.FB_SMOOTH_FREQUENCY


@dataclass(frozen=True)
class RegularizationConfig:  # regularize.hpp:19-25
    lambda_: float = 0.0
    smooth_width: int = 0
    dropout_rate: float = 0.0
    smooth_domain: SmoothDomain = SmoothDomain.TIME
    seed: int = 0

    def to_c(self) -> _lib.RegConfig:
        return _lib.RegConfig(float(self.lambda_), int(self.smooth_width), float(self.dropout_rate),
                              int(self.smooth_domain), int(self.seed) & (2**64 - 1))


_DT = {torch.float32: _lib.FB_F32, torch.bfloat16: _lib.FB_BF16, torch.float16: _lib.FB_F16}


def _stream(device: torch.device | None = None) -> C.c_void_p:
    """The current torch stream of `device` (the plan's device, not whichever
    device happens to be current)."""
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


_PREP_IDS = iter(range(1, 1 << 62))


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


class LongConvPlan:
    """Owns an ``fb_plan``: per-head spectra, twiddles and the regularized bank."""

    def __init__(self, N: int, H: int, mode: ConvMode = ConvMode.CAUSAL,
                 dtype: torch.dtype = torch.float32, engine: Engine = Engine.AUTO,
                 device: int | torch.device | None = None):
        if dtype not in _DT:
            raise TypeError(f"unsupported I/O dtype {dtype}")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if dev.type != "cuda":
            raise RuntimeError("LongConvPlan needs a CUDA device (no CPU fallback)")
        self.N, self.H, self.mode, self.dtype = int(N), int(H), ConvMode(mode), dtype
        self.device = dev
        h = C.c_void_p()
        with torch.cuda.device(dev):
            check(_lib.lib().fb_plan_create(C.byref(h), self.N, self.H, int(mode), _DT[dtype],
                                            int(engine), dev.index or 0))
        self._h = h
        info = _lib.PlanInfo()
        check(_lib.lib().fb_plan_get_info(h, C.byref(info)))
        self.n, self.l, self.m, self.engine = info.n, info.l, info.m, Engine(info.engine)
        self.tensor_cores = bool(info.tensor_cores)
        self._token = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().fb_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- K1 ------------------------------------------------------------------
    def prep(self, K: torch.Tensor, D: torch.Tensor, cfg: RegularizationConfig,
             training: bool = False) -> None:
        """regularize_bank + kernel spectrum (fb_kernel_prep)."""
        if K.shape != (self.H, self.N) or D.shape != (self.H,):
            raise DimensionError(_lib.FB_ERR_DIM, "regularized_long_conv: bank dimensions must "
                                                  "match the batch")
        K = K.detach().to(self.device, torch.float32).contiguous()
        D = D.detach().to(self.device, torch.float32).contiguous()
        c = cfg.to_c()
        check(_lib.lib().fb_kernel_prep(self._h, _ptr(K), _ptr(D), C.byref(c), int(training),
                                        _stream(self.device)))
        # every prep gets a fresh id: autograd re-preps in backward whenever the
        # plan was prepared by anyone else in between (no address-reuse aliasing)
        self._token = next(_PREP_IDS)
        self._keep = (K, D)

    def kbar(self) -> torch.Tensor:
        """Copy of the plan's regularized bank Kbar [H, N] (fp32)."""
        out = torch.empty(self.H, self.N, dtype=torch.float32, device=self.device)
        check(_lib.lib().fb_plan_copy_kbar(self._h, _ptr(out), _stream(self.device)))
        return out

    def workspace(self, B: int) -> torch.Tensor:
        nbytes = _lib.lib().fb_workspace_size(self._h, int(B))
        return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.device)

    def _check_signal(self, x: torch.Tensor, name: str) -> int:
        if x.dim() != 3 or x.shape[1] != self.H or x.shape[2] != self.N:
            raise DimensionError(_lib.FB_ERR_DIM, f"{name}: expected [B, {self.H}, {self.N}], "
                                                  f"got {list(x.shape)}")
        if x.dtype != self.dtype or x.device != self.device or not x.is_contiguous():
            raise TypeError(f"{name}: expected contiguous {self.dtype} on {self.device}")
        return x.shape[0]

    # -- K2/K3 ------------------------------------------------------------------
    def saved_size(self, B: int) -> int:
        """Bytes of the forward's saved transform (0: this plan recomputes)."""
        return int(_lib.lib().fb_saved_size(self._h, int(B)))

    def forward(self, u: torch.Tensor, out: torch.Tensor | None = None,
                workspace: torch.Tensor | None = None, save: bool | torch.Tensor = False):
        """y (and, with save=True or a buffer, (y, saved) for backward(saved=...))."""
        B = self._check_signal(u, "u")
        y = torch.empty_like(u) if out is None else out
        ws = self.workspace(B) if workspace is None else workspace
        if save is False:
            check(_lib.lib().fb_fwd(self._h, _ptr(u), _ptr(y), B, _ptr(ws), _stream(self.device)))
            return y
        nbytes = self.saved_size(B)
        saved = None
        if nbytes:
            saved = save if isinstance(save, torch.Tensor) else torch.empty(
                nbytes, dtype=torch.uint8, device=self.device)
        check(_lib.lib().fb_fwd_save(self._h, _ptr(u), _ptr(y), _ptr(saved), B, _ptr(ws),
                                     _stream(self.device)))
        return y, saved

    # -- K4 ------------------------------------------------------------------
    def backward(self, dy: torch.Tensor, u: torch.Tensor | None, want_dkbar: bool = False,
                 workspace: torch.Tensor | None = None, saved: torch.Tensor | None = None,
                 out: tuple | None = None):
        """-> (du, dK, dD[, dKbar]); dK w.r.t. the raw K given to prep().  With the
        forward's `saved` transform u may be None (tensor-core plans)."""
        B = self._check_signal(dy, "dy")
        if saved is None or u is not None:
            if u is None:
                raise DimensionError(_lib.FB_ERR_DIM, "backward: u is required without saved")
            if self._check_signal(u, "u") != B:
                raise DimensionError(_lib.FB_ERR_DIM, "backward: dy and u batch mismatch")
        if out is None:
            du = torch.empty_like(dy)
            dK = torch.empty(self.H, self.N, dtype=torch.float32, device=self.device)
            dD = torch.empty(self.H, dtype=torch.float32, device=self.device)
        else:
            du, dK, dD = out
        dKbar = torch.empty_like(dK) if want_dkbar else None
        ws = self.workspace(B) if workspace is None else workspace
        check(_lib.lib().fb_bwd_saved(self._h, _ptr(dy), _ptr(u), _ptr(saved), _ptr(du), _ptr(dK),
                                      _ptr(dKbar), _ptr(dD), B, _ptr(ws), _stream(self.device)))
        return (du, dK, dD, dKbar) if want_dkbar else (du, dK, dD)


class HostRunner:
    """regularized_long_conv forward + backward on HOST tensors
    (fb_host_runner_*): heads in chunks, copies in / kernels / copies out
    overlapped on three streams.  Host tensors should be pinned."""

    def __init__(self, N: int, H: int, B: int, dtype: torch.dtype = torch.bfloat16,
                 mode: ConvMode = ConvMode.CAUSAL, engine: Engine = Engine.AUTO,
                 heads_per_chunk: int | None = None, device: int | torch.device | None = None):
        if dtype not in _DT:
            raise TypeError(f"unsupported I/O dtype {dtype}")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.N, self.H, self.B, self.dtype, self.device = int(N), int(H), int(B), dtype, dev
        hc = heads_per_chunk if heads_per_chunk else max(1, self.H // 8)
        h = C.c_void_p()
        with torch.cuda.device(dev):
            check(_lib.lib().fb_host_runner_create(C.byref(h), self.N, self.H, int(mode), _DT[dtype],
                                                   int(engine), dev.index or 0, self.B, int(hc)))
        self._h = h
        self.chunk_heads = int(_lib.lib().fb_host_runner_chunk_heads(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().fb_host_runner_destroy(h)
            except Exception:
                pass
            self._h = None

    def run(self, u, dy, K, D, cfg: RegularizationConfig, training: bool = False, out=None):
        """-> (y, du, dK, dD) host tensors; stream-ordered on the current stream."""
        B, H, N = self.B, self.H, self.N
        for x, name, shape, dt in ((u, "u", (B, H, N), self.dtype), (dy, "dy", (B, H, N), self.dtype),
                                   (K, "K", (H, N), torch.float32), (D, "D", (H,), torch.float32)):
            if tuple(x.shape) != shape or x.dtype != dt or x.is_cuda or not x.is_contiguous():
                raise DimensionError(_lib.FB_ERR_DIM, f"{name}: expected contiguous host {dt} "
                                                      f"{list(shape)}")
        if out is None:
            out = (torch.empty_like(u, pin_memory=True), torch.empty_like(u, pin_memory=True),
                   torch.empty_like(K, pin_memory=True), torch.empty_like(D, pin_memory=True))
        y, du, dK, dD = out
        c = cfg.to_c()
        with torch.cuda.device(self.device):
            check(_lib.lib().fb_host_runner_run(self._h, C.byref(c), int(training), _ptr(u), _ptr(dy),
                                                _ptr(K), _ptr(D), _ptr(y), _ptr(du), _ptr(dK),
                                                _ptr(dD), _stream(self.device)))
        return y, du, dK, dD


class InitKind(enum.IntEnum):  # regularize.hpp:27
    RANDOM = 0
    GEOMETRIC = 1


def init_kernels(kind: InitKind, H: int, N: int, seed: int, device=None,
                 dtype: torch.dtype = torch.float32) -> tuple[torch.Tensor, torch.Tensor]:
    """init_kernels (regularize.hpp:55, regularize.cpp:73-91) on the device:
    the reference's RNG streams exactly (K[h] from child stream h, D from child
    stream H).  Returns (K [H, N], D [H]) in fp32 or fp64."""
    if H < 1 or N < 1:
        raise DimensionError(_lib.FB_ERR_DIM, "init_kernels: heads and len must be >= 1")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    K = torch.empty(H, N, dtype=dtype, device=dev)
    D = torch.empty(H, dtype=dtype, device=dev)
    f64 = dtype == torch.float64
    with torch.cuda.device(dev):
        check(_lib.lib().fb_init_kernels(int(kind), int(H), int(N), int(seed) & (2**64 - 1),
                                         _ptr(None if f64 else K), _ptr(None if f64 else D),
                                         _ptr(K if f64 else None), _ptr(D if f64 else None),
                                         dev.index or 0, _stream(dev)))
    return K, D


_PLANS: dict = {}


def get_plan(N: int, H: int, mode: ConvMode, dtype: torch.dtype, engine: Engine,
             device: torch.device) -> LongConvPlan:
    key = (N, H, int(mode), dtype, int(engine), str(device))
    p = _PLANS.get(key)
    if p is None:
        p = LongConvPlan(N, H, mode, dtype, engine, device)
        _PLANS[key] = p
    return p


def regularized_long_conv(u: torch.Tensor, K: torch.Tensor, D: torch.Tensor,
                          cfg: RegularizationConfig = RegularizationConfig(),
                          engine: Engine = Engine.AUTO, mode: ConvMode = ConvMode.CAUSAL,
                          training: bool = False) -> torch.Tensor:
    """y[b,h] = conv(u[b,h], regularize(K)[h]) + D[h] u[b,h] (regularize.hpp:67-70).
    ``threads`` of the reference has no meaning here (the grid is the parallelism)."""
    if u.dim() != 3:
        raise DimensionError(_lib.FB_ERR_DIM, "regularized_long_conv: u must be [B, H, N]")
    B, H, N = u.shape
    plan = get_plan(N, H, mode, u.dtype, engine, u.device)
    plan.prep(K, D, cfg, training)
    return plan.forward(u.contiguous())


def regularized_long_conv_backward(dy: torch.Tensor, u: torch.Tensor, K: torch.Tensor,
                                   D: torch.Tensor,
                                   cfg: RegularizationConfig = RegularizationConfig(),
                                   engine: Engine = Engine.AUTO,
                                   mode: ConvMode = ConvMode.CAUSAL, training: bool = False,
                                   want_dkbar: bool = False):
    """(du, dK, dD[, dKbar]) for the layer above (SURVEY.md §8c formulas)."""
    B, H, N = u.shape
    plan = get_plan(N, H, mode, u.dtype, engine, u.device)
    plan.prep(K, D, cfg, training)
    return plan.backward(dy.contiguous(), u.contiguous(), want_dkbar)


class _LongConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, u, K, D, cfg, engine, mode, training):
        B, H, N = u.shape
        plan = get_plan(N, H, mode, u.dtype, engine, u.device)
        plan.prep(K, D, cfg, training)
        # tensor-core plans also keep the forward's transform of u (the
        # backward then skips recomputing it)
        y, saved = plan.forward(u.contiguous(), save=True)
        ctx.save_for_backward(u, K, D)
        ctx.saved_u = saved
        ctx.cfg, ctx.plan, ctx.training = cfg, plan, training
        ctx.token = plan._token
        return y

    @staticmethod
    def backward(ctx, dy):
        u, K, D = ctx.saved_tensors
        plan = ctx.plan
        if plan._token != ctx.token:  # plan re-prepared by another call meanwhile
            plan.prep(K, D, ctx.cfg, ctx.training)
        du, dK, dD = plan.backward(dy.contiguous().to(u.dtype), u.contiguous(), saved=ctx.saved_u)
        ctx.saved_u = None
        return du, dK.to(K.dtype), dD.to(D.dtype), None, None, None, None


def long_conv(u: torch.Tensor, K: torch.Tensor, D: torch.Tensor,
              cfg: RegularizationConfig = RegularizationConfig(), engine: Engine = Engine.AUTO,
              mode: ConvMode = ConvMode.CAUSAL, training: bool = False) -> torch.Tensor:
    """Differentiable regularized long convolution (Algorithm 1)."""
    return _LongConvFn.apply(u, K, D, cfg, engine, mode, training)

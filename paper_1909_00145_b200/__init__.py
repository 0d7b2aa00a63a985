"""B200-native stochastic spatial-domain CSC hot path (arxiv 1909.00145).

Thin Python binding over the C ABI in include/csc.h (libcsc_b200.so, built with
nvcc for sm_100a).  Argument marshalling only: every step of the path runs in
the library's CUDA kernels.  There is NO CPU fallback: if the extension is
missing or no B200 is visible, construction fails loudly.

PyTorch is used for device memory and streams only.  Tensors passed in must be
contiguous float32 CUDA tensors in the layouts of include/csc.h:
  x [n_local, H, W], d [K, s, s], z [n_local, K, H+s-1, W+s-1].
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcsc_b200.so")

CSC_OK = 0
_STATUS = {0: "CSC_OK", 1: "CSC_ERR_ARG", 2: "CSC_ERR_SHAPE", 3: "CSC_ERR_CUDA", 4: "CSC_ERR_NCCL",
           5: "CSC_ERR_OOM", 6: "CSC_ERR_NONFINITE"}

# Every symbol include/csc.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = (
    "csc_init", "csc_code_step", "csc_filter_step", "csc_objective", "csc_iterate", "csc_invalidate",
    "csc_zero_codes", "csc_destroy", "csc_last_error", "csc_nccl_unique_id", "csc_abi_version",
    "csc_mask_bits", "csc_read_residual", "csc_read_grad", "csc_lipschitz", "csc_launch_count",
    "csc_profile_enable", "csc_profile_read", "csc_kernel_variants", "csc_code_step_admm",
    "csc_set_step_rule", "csc_read_step_z", "csc_filter_step_bcd", "csc_surrogate_reset",
    "csc_surrogate_update", "csc_filter_step_surrogate", "csc_read_surrogate", "csc_set_mask_mode",
    "csc_stage_images", "csc_iterate_staged", "csc_mask_selwords", "csc_read_scalars", "csc_zg_sumsq",
    "csc_set_iter_offset", "csc_count_nonzero", "csc_set_nvtx", "csc_comm_check", "csc_profile_set_classes",
    "csc_objective_enqueue", "csc_objective_read", "csc_profile_sample", "csc_iterate_staged_async",
    "csc_iterate_drain", "csc_load_staged",
)

# csc_kernel_class (include/csc.h)
KERNEL_CLASSES = ("conv", "conv_finalize", "wgrad", "code_step", "mask", "lipschitz", "small", "admm", "bcd")


class CSCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Dims(ctypes.Structure):
    _fields_ = [("n_local", ctypes.c_int32), ("K", ctypes.c_int32), ("s", ctypes.c_int32),
                ("H", ctypes.c_int32), ("W", ctypes.c_int32), ("world", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("nccl_id", ctypes.c_void_p)]


_lib = None
_lib_lock = threading.Lock()


def load_library(path: Optional[str] = None):
    """Load libcsc_b200.so (raises if it is missing -- build with __graft_entry__.build())."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        # CSC_LIB_PATH: load another build of the same library (side-by-side A/B timing of two builds)
        p = path or os.environ.get("CSC_LIB_PATH") or LIB_PATH
        if not os.path.exists(p):
            raise ImportError(f"{p} not found: the CUDA extension is not built "
                              "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        L = ctypes.CDLL(p)
        vp, f32, f64, u32, u64 = ctypes.c_void_p, ctypes.c_float, ctypes.c_double, ctypes.c_uint32, ctypes.c_uint64
        L.csc_init.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(vp)]
        L.csc_code_step.argtypes = [vp, vp, vp, vp, f32, f32, f64, u64, u32, vp]
        L.csc_filter_step.argtypes = [vp, vp, vp, vp, f32, vp]
        L.csc_set_step_rule.argtypes = [vp, ctypes.c_int]
        L.csc_set_mask_mode.argtypes = [vp, ctypes.c_int]
        L.csc_stage_images.argtypes = [vp, vp, ctypes.c_int]
        L.csc_iterate_staged.argtypes = [vp, ctypes.c_int, vp, vp, vp, f32, f32, f32, f64, u64, u32, vp, vp]
        L.csc_iterate_staged_async.argtypes = [vp, ctypes.c_int, vp, vp, vp, f32, f32, f32, f64, u64, u32, vp, vp, vp]
        L.csc_iterate_drain.argtypes = [vp, vp, vp, vp]
        L.csc_load_staged.argtypes = [vp, ctypes.c_int, vp]
        L.csc_filter_step_bcd.argtypes = [vp, vp, vp, vp, ctypes.c_int, vp]
        L.csc_surrogate_reset.argtypes = [vp]
        L.csc_surrogate_update.argtypes = [vp, vp, vp]
        L.csc_filter_step_surrogate.argtypes = [vp, vp, ctypes.c_int, vp]
        L.csc_read_surrogate.argtypes = [vp, vp, vp, ctypes.POINTER(ctypes.c_int64)]
        L.csc_read_step_z.argtypes = [vp, vp]
        L.csc_code_step_admm.argtypes = [vp, vp, vp, vp, f32, f32, f32, ctypes.c_int, ctypes.c_int, f64, u64, u32]
        L.csc_objective.argtypes = [vp, vp, vp, vp, f32, vp]
        L.csc_iterate.argtypes = [vp, vp, vp, vp, vp, f32, f32, f32, f64, u64, u32, vp, vp]
        L.csc_invalidate.argtypes = [vp]
        L.csc_zero_codes.argtypes = [vp, vp, vp]
        L.csc_destroy.argtypes = [vp]
        L.csc_last_error.argtypes = [vp]
        L.csc_last_error.restype = ctypes.c_char_p
        L.csc_nccl_unique_id.argtypes = [vp]
        L.csc_abi_version.restype = ctypes.c_int
        L.csc_mask_bits.argtypes = [vp, u32, f64, u64, vp]
        L.csc_mask_selwords.argtypes = [vp, u32, f64, u64, vp, vp]
        L.csc_read_scalars.argtypes = [vp, vp]
        L.csc_set_iter_offset.argtypes = [vp, vp]
        L.csc_zg_sumsq.argtypes = [vp, vp, vp]
        L.csc_read_residual.argtypes = [vp, vp]
        L.csc_read_grad.argtypes = [vp, vp]
        L.csc_lipschitz.argtypes = [vp, vp, vp]
        L.csc_count_nonzero.argtypes = [vp, vp, ctypes.c_int64, ctypes.POINTER(u64)]
        L.csc_set_nvtx.argtypes = [vp, ctypes.c_int]
        L.csc_comm_check.argtypes = [vp]
        L.csc_launch_count.argtypes = [vp]
        L.csc_launch_count.restype = u64
        L.csc_profile_enable.argtypes = [vp, ctypes.c_int]
        L.csc_profile_set_classes.argtypes = [vp, u32]
        L.csc_profile_sample.argtypes = [vp]
        L.csc_objective_enqueue.argtypes = [vp, vp, vp, vp]
        L.csc_objective_read.argtypes = [vp, f32, vp]
        L.csc_profile_read.argtypes = [vp, ctypes.c_int, ctypes.POINTER(f64), ctypes.POINTER(u64)]
        L.csc_kernel_variants.argtypes = [vp]
        L.csc_kernel_variants.restype = u32
        for name in ABI_SYMBOLS:
            if name not in ("csc_last_error", "csc_abi_version", "csc_launch_count", "csc_kernel_variants"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
        return L


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = (ctypes.c_uint8 * 128)()
    st = L.csc_nccl_unique_id(buf)
    if st != CSC_OK:
        raise CSCError(st, L.csc_last_error(None).decode())
    return bytes(buf)


def _ptr(t, name: str, numel: Optional[int] = None) -> int:
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")
    return t.data_ptr()


class Context:
    """One csc_ctx: (rank, device, stream).  See include/csc.h for semantics."""

    def __init__(self, n_local: int, K: int, s: int, H: int, W: int, *, world: int = 1, rank: int = 0,
                 device: Optional[int] = None, stream=None, nccl_id: Optional[bytes] = None):
        import torch
        self._L = load_library()
        if device is None:
            device = torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self.n_local, self.K, self.s, self.H, self.W = n_local, K, s, H, W
        self.Hc, self.Wc = H + s - 1, W + s - 1
        self.world, self.rank, self.device = world, rank, device
        self._idbuf = None
        if nccl_id is not None:
            self._idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        dims = _Dims(n_local, K, s, H, W, world, rank, device, ctypes.c_void_p(stream.cuda_stream),
                     ctypes.cast(self._idbuf, ctypes.c_void_p) if self._idbuf is not None else None)
        h = ctypes.c_void_p()
        st = self._L.csc_init(ctypes.byref(dims), ctypes.byref(h))
        if st != CSC_OK:
            raise CSCError(st, self._L.csc_last_error(None).decode())
        self._h = h

    # -- helpers
    def _check(self, st: int):
        if st != CSC_OK:
            raise CSCError(st, self._L.csc_last_error(self._h).decode())

    def _xdz(self, x, d, z):
        nx = self.n_local * self.H * self.W
        nz = self.n_local * self.K * self.Hc * self.Wc
        return (_ptr(x, "x", nx) if self.n_local else 0, _ptr(d, "d", self.K * self.s * self.s),
                _ptr(z, "z", nz) if self.n_local else 0)

    # -- ABI
    def code_step(self, x, d, z, lam: float, p: float, seed: int, it: int, step_z: float = 0.0,
                  want_step: bool = False) -> Optional[float]:
        px, pd, pz = self._xdz(x, d, z)
        out = ctypes.c_float(0.0)
        self._check(self._L.csc_code_step(self._h, px, pd, pz, float(lam), float(step_z), float(p),
                                          int(seed) & (2**64 - 1), int(it) & 0xffffffff,
                                          ctypes.byref(out) if want_step else None))
        return float(out.value) if want_step else None

    def filter_step_bcd(self, x, d, z, sweeps: int = 1, want_flags: bool = False):
        """Projected block-coordinate filter update (include/csc.h csc_filter_step_bcd).
        Returns the K per-filter flags (1 = left unchanged) when want_flags."""
        px, pd, pz = self._xdz(x, d, z)
        flags = (ctypes.c_uint8 * max(self.K, 1))()
        self._check(self._L.csc_filter_step_bcd(self._h, px, pd, pz, int(sweeps),
                                                ctypes.cast(flags, ctypes.c_void_p) if want_flags else None))
        return list(flags)[:self.K] if want_flags else None

    def surrogate_reset(self) -> None:
        """Online surrogates C = 0, B = 0, t = 0 (include/csc.h csc_surrogate_reset; Eq.7)."""
        self._check(self._L.csc_surrogate_reset(self._h))

    def surrogate_update(self, x, z) -> None:
        """Fold the mini-batch (x, z) into C, B (Eq.7)."""
        nx = self.n_local * self.H * self.W
        nz = self.n_local * self.K * self.Hc * self.Wc
        self._check(self._L.csc_surrogate_update(self._h, _ptr(x, "x", nx) if self.n_local else 0,
                                                 _ptr(z, "z", nz) if self.n_local else 0))

    def filter_step_surrogate(self, d, sweeps: int = 1, want_flags: bool = False):
        """Eq.8 projected block-coordinate filter update on the surrogates."""
        flags = (ctypes.c_uint8 * max(self.K, 1))()
        self._check(self._L.csc_filter_step_surrogate(self._h, _ptr(d, "d", self.K * self.s * self.s), int(sweeps),
                                                      ctypes.cast(flags, ctypes.c_void_p) if want_flags else None))
        return list(flags)[:self.K] if want_flags else None

    def read_surrogate(self, C, B) -> int:
        """Copy C [K][K][M][M] and B [K][M] (float64 CUDA tensors) and return t."""
        import torch
        M = self.s * self.s
        for t_, n_, nm in ((C, self.K * self.K * M * M, "C"), (B, self.K * M, "B")):
            if not (t_.is_cuda and t_.dtype == torch.float64 and t_.is_contiguous() and t_.numel() == n_):
                raise ValueError(f"{nm} must be a contiguous float64 CUDA tensor with {n_} elements")
        t = ctypes.c_int64(0)
        self._check(self._L.csc_read_surrogate(self._h, C.data_ptr(), B.data_ptr(), ctypes.byref(t)))
        return int(t.value)

    MASK_MODES = {"entry": 0, "sector8": 1}

    def set_mask_mode(self, mode: str) -> None:
        """Mask sampling: "entry" (Eq.2, default) or "sector8" (one draw per 8-code block; a labelled
        deviation, include/csc.h csc_set_mask_mode)."""
        self._check(self._L.csc_set_mask_mode(self._h, self.MASK_MODES[mode]))

    STEP_RULES = {"lipschitz": 0, "eso": 1}

    def set_step_rule(self, rule: str) -> None:
        """Built-in tau_z rule when step_z == 0: "lipschitz" (1/L_D) or "eso" (per filter,
        include/csc.h csc_set_step_rule)."""
        self._check(self._L.csc_set_step_rule(self._h, self.STEP_RULES[rule]))

    def read_step_z(self, out) -> None:
        """K step sizes of the last code step into the float32 CUDA tensor out."""
        self._check(self._L.csc_read_step_z(self._h, _ptr(out, "out", self.K)))

    def code_step_admm(self, x, d, z, lam: float, p: float, seed: int, it: int, rho: float = 0.0,
                       alpha: float = 1.8, n_admm: int = 10, n_cg: int = 5) -> None:
        """ADMM masked-LASSO code update (include/csc.h csc_code_step_admm)."""
        px, pd, pz = self._xdz(x, d, z)
        self._check(self._L.csc_code_step_admm(self._h, px, pd, pz, float(lam), float(rho), float(alpha),
                                               int(n_admm), int(n_cg), float(p), int(seed) & (2**64 - 1),
                                               int(it) & 0xffffffff))

    def filter_step(self, x, d, z, step_d: float = 0.0, want_step: bool = False) -> Optional[float]:
        px, pd, pz = self._xdz(x, d, z)
        out = ctypes.c_float(0.0)
        self._check(self._L.csc_filter_step(self._h, px, pd, pz, float(step_d),
                                            ctypes.byref(out) if want_step else None))
        return float(out.value) if want_step else None

    def objective(self, x, d, z, lam: float) -> Tuple[float, float, float]:
        px, pd, pz = self._xdz(x, d, z)
        out = (ctypes.c_double * 3)()
        self._check(self._L.csc_objective(self._h, px, pd, pz, float(lam), out))
        return float(out[0]), float(out[1]), float(out[2])

    def objective_enqueue(self, x, d, z) -> None:
        """The objective pass without synchronising (csc_objective_enqueue; capturable in a CUDA graph)."""
        px, pd, pz = self._xdz(x, d, z)
        self._check(self._L.csc_objective_enqueue(self._h, px, pd, pz))

    def objective_read(self, lam: float) -> Tuple[float, float, float]:
        """(F, fit, l1) of the last enqueued objective pass (csc_objective_read; syncs)."""
        out = (ctypes.c_double * 3)()
        self._check(self._L.csc_objective_read(self._h, float(lam), out))
        return float(out[0]), float(out[1]), float(out[2])

    def iterate(self, x, d, z, lam: float, p: float, seed: int, it: int, *, x_host=None,
                step_z: float = 0.0, step_d: float = 0.0):
        """One SBCSC iteration (code step, filter step, objective).  x_host: optional pinned CPU
        float32 tensor uploaded into x first.  Returns ((F, fit, l1), (tau_z, tau_d))."""
        px, pd, pz = self._xdz(x, d, z)
        ph = None
        if x_host is not None:
            if x_host.is_cuda or x_host.dtype.itemsize != 4 or not x_host.is_contiguous():
                raise ValueError("x_host must be a contiguous float32 CPU tensor")
            if x_host.numel() != self.n_local * self.H * self.W:
                raise ValueError("x_host has the wrong size")
            ph = x_host.data_ptr()
        obj = (ctypes.c_double * 3)()
        taus = (ctypes.c_float * 2)()
        self._check(self._L.csc_iterate(self._h, ph, px, pd, pz, float(lam), float(step_z), float(step_d),
                                        float(p), int(seed) & (2**64 - 1), int(it) & 0xffffffff, obj, taus))
        return (float(obj[0]), float(obj[1]), float(obj[2])), (float(taus[0]), float(taus[1]))

    def stage_images(self, x_host, slot: int) -> None:
        """Asynchronous copy of the pinned CPU float32 tensor x_host into staging slot 0/1
        (include/csc.h csc_stage_images); x_host must stay alive until the copy has run."""
        if x_host.is_cuda or x_host.dtype.itemsize != 4 or not x_host.is_contiguous():
            raise ValueError("x_host must be a contiguous float32 CPU tensor")
        if x_host.numel() != self.n_local * self.H * self.W:
            raise ValueError("x_host has the wrong size")
        self._check(self._L.csc_stage_images(self._h, x_host.data_ptr(), int(slot)))

    def iterate_staged(self, x, d, z, lam: float, p: float, seed: int, it: int, slot: int, *, step_z: float = 0.0,
                       step_d: float = 0.0):
        """csc_iterate with the images of a staged slot (include/csc.h csc_iterate_staged)."""
        px, pd, pz = self._xdz(x, d, z)
        obj = (ctypes.c_double * 3)()
        taus = (ctypes.c_float * 2)()
        self._check(self._L.csc_iterate_staged(self._h, int(slot), px, pd, pz, float(lam), float(step_z),
                                               float(step_d), float(p), int(seed) & (2**64 - 1),
                                               int(it) & 0xffffffff, obj, taus))
        return (float(obj[0]), float(obj[1]), float(obj[2])), (float(taus[0]), float(taus[1]))

    def iterate_staged_async(self, x, d, z, lam: float, p: float, seed: int, it: int, slot: int, *,
                             step_z: float = 0.0, step_d: float = 0.0):
        """Pipelined csc_iterate_staged (include/csc.h csc_iterate_staged_async): enqueues this iteration
        and returns the previous call's ((F, 1/2||r||^2, lambda||z||_1), (tau_z, tau_d)), or None."""
        px, pd, pz = self._xdz(x, d, z)
        obj = (ctypes.c_double * 3)()
        taus = (ctypes.c_float * 2)()
        have = ctypes.c_int(0)
        self._check(self._L.csc_iterate_staged_async(self._h, int(slot), px, pd, pz, float(lam), float(step_z),
                                                     float(step_d), float(p), int(seed) & (2**64 - 1),
                                                     int(it) & 0xffffffff, obj, taus, ctypes.byref(have)))
        if not have.value:
            return None
        return (float(obj[0]), float(obj[1]), float(obj[2])), (float(taus[0]), float(taus[1]))

    def load_staged(self, x, slot: int):
        """Enqueue the images of a staged slot into x (and move the residual cache), capturable
        (include/csc.h csc_load_staged)."""
        self._check(self._L.csc_load_staged(self._h, int(slot),
                                            _ptr(x, "x", self.n_local * self.H * self.W) if self.n_local else 0))

    def iterate_drain(self):
        """The results of the last csc_iterate_staged_async call (include/csc.h csc_iterate_drain), or None."""
        obj = (ctypes.c_double * 3)()
        taus = (ctypes.c_float * 2)()
        have = ctypes.c_int(0)
        self._check(self._L.csc_iterate_drain(self._h, obj, taus, ctypes.byref(have)))
        if not have.value:
            return None
        return (float(obj[0]), float(obj[1]), float(obj[2])), (float(taus[0]), float(taus[1]))

    def invalidate(self):
        self._check(self._L.csc_invalidate(self._h))

    def zero_codes(self, x, z):
        px = _ptr(x, "x") if self.n_local else 0
        pz = _ptr(z, "z") if self.n_local else 0
        self._check(self._L.csc_zero_codes(self._h, px, pz))

    def mask_bits(self, it: int, p: float, seed: int, out):
        import torch
        nwords = (self.K * self.Hc * self.Wc + 31) // 32
        if not (out.is_cuda and out.dtype == torch.int32 and out.numel() == nwords and out.is_contiguous()):
            raise ValueError(f"out must be a contiguous int32 CUDA tensor of {nwords} words")
        self._check(self._L.csc_mask_bits(self._h, int(it) & 0xffffffff, float(p), int(seed) & (2**64 - 1),
                                          out.data_ptr()))

    def mask_selwords(self, it: int, p: float, seed: int, out=None):
        """The selection words of the tensor-core code step (csc_mask_selwords); returns
        (nkg, wper, wnc, KC).  out: contiguous int32 CUDA tensor of nkg*wper*Hc*Wc words, or None."""
        info = (ctypes.c_int32 * 4)()
        self._check(self._L.csc_mask_selwords(self._h, 0, 1.0, 0, None, info))
        if out is not None:
            import torch
            n = info[0] * info[1] * self.Hc * self.Wc
            if not (out.is_cuda and out.dtype == torch.int32 and out.numel() == n and out.is_contiguous()):
                raise ValueError(f"out must be a contiguous int32 CUDA tensor of {n} words")
            self._check(self._L.csc_mask_selwords(self._h, int(it) & 0xffffffff, float(p), int(seed) & (2**64 - 1),
                                                  out.data_ptr(), info))
        return tuple(info)

    def set_iter_offset(self, offset) -> None:
        """Mask iteration = iter + offset[0] read on the device (include/csc.h csc_set_iter_offset);
        offset: int32 CUDA tensor of 1 element kept alive by the caller, or None to clear."""
        import torch
        if offset is None:
            self._check(self._L.csc_set_iter_offset(self._h, None))
            return
        if not (offset.is_cuda and offset.dtype == torch.int32 and offset.numel() >= 1):
            raise ValueError("offset must be an int32 CUDA tensor")
        self._iter_off = offset
        self._check(self._L.csc_set_iter_offset(self._h, offset.data_ptr()))

    def read_scalars(self) -> dict:
        """Device scalars after the last steps (include/csc.h csc_read_scalars)."""
        out = (ctypes.c_double * 4)()
        self._check(self._L.csc_read_scalars(self._h, out))
        return {"sum_r2": out[0], "l1": out[1], "zg2": out[2], "gg": out[3]}

    def zg_sumsq(self, z, g) -> float:
        """||sum_k g_k * z_k||^2 over this context's images for a float64 CUDA tensor g [K*s*s]."""
        import torch
        if not (g.is_cuda and g.dtype == torch.float64 and g.numel() == self.K * self.s * self.s):
            raise ValueError("g must be a float64 CUDA tensor of K*s*s elements")
        nz = self.n_local * self.K * self.Hc * self.Wc
        self._check(self._L.csc_zg_sumsq(self._h, _ptr(z, "z", nz) if self.n_local else 0, g.data_ptr()))
        return self.read_scalars()["zg2"]

    def read_residual(self, out):
        self._check(self._L.csc_read_residual(self._h, _ptr(out, "out", self.n_local * self.H * self.W)
                                              if self.n_local else 0))

    def read_grad(self, out):
        import torch
        if not (out.is_cuda and out.dtype == torch.float64 and out.numel() == self.K * self.s * self.s):
            raise ValueError("out must be a float64 CUDA tensor of K*s*s elements")
        self._check(self._L.csc_read_grad(self._h, out.data_ptr()))

    def lipschitz(self, d) -> float:
        out = ctypes.c_double(0.0)
        self._check(self._L.csc_lipschitz(self._h, _ptr(d, "d"), ctypes.byref(out)))
        return float(out.value)

    def count_nonzero(self, v) -> int:
        """Number of nonzero entries of a float32 CUDA tensor (include/csc.h csc_count_nonzero; syncs)."""
        n = ctypes.c_uint64(0)
        numel = int(v.numel())
        self._check(self._L.csc_count_nonzero(self._h, _ptr(v, "v") if numel else None, numel, ctypes.byref(n)))
        return int(n.value)

    def set_nvtx(self, on: bool = True):
        """NVTX ranges around every entry point of this context (csc_set_nvtx)."""
        self._check(self._L.csc_set_nvtx(self._h, 1 if on else 0))

    def comm_check(self):
        """Raise CSCError if the NCCL communicator reports an asynchronous error (csc_comm_check)."""
        self._check(self._L.csc_comm_check(self._h))

    def profile_enable(self, on: bool = True, classes=None):
        """Per-launch event timing on (resets the totals); classes: names from KERNEL_CLASSES to time
        (None: all) -- csc_profile_set_classes."""
        mask = 0xFFFFFFFF if classes is None else sum(1 << KERNEL_CLASSES.index(c) for c in classes)
        self._check(self._L.csc_profile_set_classes(self._h, mask))
        self._check(self._L.csc_profile_enable(self._h, 1 if on else 0))

    def profile_sample(self) -> None:
        """Accumulate the recorded event pairs and keep them (csc_profile_sample: after graph replays)."""
        self._check(self._L.csc_profile_sample(self._h))

    def profile_read(self) -> dict:
        """{class: (total_ms, launches)} accumulated since profile_enable(True) (syncs)."""
        out = {}
        for i, name in enumerate(KERNEL_CLASSES):
            ms, n = ctypes.c_double(0.0), ctypes.c_uint64(0)
            self._check(self._L.csc_profile_read(self._h, i, ctypes.byref(ms), ctypes.byref(n)))
            out[name] = (float(ms.value), int(n.value))
        return out

    @property
    def tc_dense(self) -> bool:
        """True when the dense passes run on the tcgen05 3xTF32 kernel (csc_kernel_variants bit 0)."""
        return bool(self._L.csc_kernel_variants(self._h) & 1)

    @property
    def tc_wgrad(self) -> bool:
        """True when the filter gradient runs on the tcgen05 3xTF32 kernel (csc_kernel_variants bit 1)."""
        return bool(self._L.csc_kernel_variants(self._h) & 2)

    @property
    def variants(self) -> int:
        """csc_kernel_variants bit set (include/csc.h)."""
        return int(self._L.csc_kernel_variants(self._h))

    @property
    def tc_code(self) -> bool:
        """True when the masked code step runs as the tcgen05 dense-then-mask kernel (bit 2)."""
        return bool(self._L.csc_kernel_variants(self._h) & 4)

    @property
    def launch_count(self) -> int:
        return int(self._L.csc_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.csc_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


__all__: Sequence[str] = ["Context", "CSCError", "load_library", "nccl_unique_id", "LIB_PATH", "ABI_SYMBOLS"]

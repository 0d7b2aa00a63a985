"""ctypes wrapper of the CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product path
(paper_1909_00145_b200/) never imports it and shares no code with it.

Every function takes/returns numpy arrays in the layouts of include/csc.h:
x[N][H][W], d[K][s][s], z[N][K][H+s-1][W+s-1] (C-contiguous).  dtype float32
selects the fp32-state oracle (parity with the GPU), float64 the exact-arithmetic
build used by the pins.  Sums always accumulate in fp64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_c_i64 = ctypes.c_int64
_c_dbl = ctypes.c_double
_c_u64 = ctypes.c_uint64
_c_u32 = ctypes.c_uint32
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile liboracle.so with the oracle's own Makefile (g++ -O2 -fopenmp)."""
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            L.oracle_num_threads.restype = ctypes.c_int
            L.oracle_philox4x32_10.argtypes = [_vp, _vp, _vp]
            L.oracle_philox_batch.argtypes = [_c_i64, _vp, _vp, _vp]
            L.oracle_mask_threshold.argtypes = [_c_dbl]
            L.oracle_mask_threshold.restype = _c_u64
            L.oracle_mask_bits.argtypes = [_c_i64, _c_i64, _c_i64, _c_dbl, _c_u64, _c_u32, _vp]
            L.oracle_mask_bits_mode.argtypes = [_c_i64, _c_i64, _c_i64, _c_dbl, _c_u64, _c_u32, _vp, ctypes.c_int]
            L.oracle_soft_threshold.argtypes = [_c_dbl, _c_dbl]
            L.oracle_soft_threshold.restype = _c_dbl
            for suf in ("f32", "f64"):
                getattr(L, f"oracle_residual_{suf}").argtypes = [_c_i64] * 5 + [_vp] * 4
                getattr(L, f"oracle_dtr_{suf}").argtypes = [_c_i64] * 5 + [_vp] * 3
                getattr(L, f"oracle_filter_grad_{suf}").argtypes = [_c_i64] * 5 + [_vp] * 3
                f = getattr(L, f"oracle_lipschitz_{suf}")
                f.argtypes = [_c_i64, _c_i64, _vp]
                f.restype = _c_dbl
                getattr(L, f"oracle_code_step_{suf}").argtypes = (
                    [_c_i64] * 5 + [_vp] * 3 + [_c_dbl, _c_dbl, _c_dbl, _c_u64, _c_u32, _vp, ctypes.c_int,
                                                ctypes.c_int])
                getattr(L, f"oracle_admm_code_step_{suf}").argtypes = (
                    [_c_i64] * 5 + [_vp] * 3 + [_c_dbl, _c_dbl, _c_dbl, ctypes.c_int, ctypes.c_int, _c_dbl, _c_u64,
                                                _c_u32])
                getattr(L, f"oracle_filter_step_{suf}").argtypes = (
                    [_c_i64] * 5 + [_vp] * 3 + [_c_dbl, _vp, _vp, _vp])
                getattr(L, f"oracle_objective_{suf}").argtypes = [_c_i64] * 5 + [_vp] * 3 + [_c_dbl, _vp]
                getattr(L, f"oracle_filter_step_bcd_{suf}").argtypes = (
                    [_c_i64] * 5 + [_vp] * 3 + [ctypes.c_int, _vp])
                getattr(L, f"oracle_surrogate_update_{suf}").argtypes = [_c_i64] * 5 + [_vp] * 4 + [_c_i64]
                getattr(L, f"oracle_filter_step_surrogate_{suf}").argtypes = [_c_i64] * 2 + [_vp] * 3 + [
                    ctypes.c_int, _vp]
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _suf(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise TypeError(f"oracle supports float32/float64 state, got {dt}")


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def philox4x32_10(ctr, key) -> np.ndarray:
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.empty_like(ctr)
    lib().oracle_philox_batch(ctr.shape[0], _p(ctr), _p(key), _p(out))
    return out


def mask_threshold(p: float) -> int:
    return int(lib().oracle_mask_threshold(float(p)))


MASK_MODES = {"entry": 0, "sector8": 1}


def mask_bits(K: int, Hc: int, Wc: int, p: float, seed: int, t: int, mode: str = "entry") -> np.ndarray:
    """Canonical mask bits; mode "sector8": one draw per aligned block of 8 coordinates (E5)."""
    total = K * Hc * Wc
    out = np.zeros((total + 31) // 32, dtype=np.uint32)
    if mode == "entry":
        lib().oracle_mask_bits(K, Hc, Wc, float(p), int(seed) & (2**64 - 1), int(t) & 0xffffffff, _p(out))
    else:
        lib().oracle_mask_bits_mode(K, Hc, Wc, float(p), int(seed) & (2**64 - 1), int(t) & 0xffffffff, _p(out),
                                    MASK_MODES[mode])
    return out


def unpack_mask(bits: np.ndarray, K: int, Hc: int, Wc: int) -> np.ndarray:
    """Bool mask [K][Hc][Wc] from the ABI bit layout (bit l of word l>>5, LSB first)."""
    b = np.unpackbits(bits.view(np.uint8), bitorder="little")[: K * Hc * Wc]
    return b.reshape(K, Hc, Wc).astype(bool)


def soft_threshold(w: float, kappa: float) -> float:
    return float(lib().oracle_soft_threshold(float(w), float(kappa)))


def residual(x, d, z, dtype=np.float32) -> np.ndarray:
    """r = sum_k d_k * z_k - x (valid true convolution).  x may be None (-> Dz)."""
    d = _c(d, dtype); z = _c(z, dtype)
    N, K, Hc, Wc = z.shape
    s = d.shape[-1]
    H, W = Hc - s + 1, Wc - s + 1
    xx = _c(x, dtype) if x is not None else None
    r = np.empty((N, H, W), dtype=dtype)
    getattr(lib(), f"oracle_residual_{_suf(dtype)}")(N, K, s, H, W, _p(xx) if xx is not None else None,
                                                   _p(d), _p(z), _p(r))
    return r


def dtr(d, r, dtype=np.float64) -> np.ndarray:
    """D^T r for all codes: out[n,k,u,v] = sum_ab d[k,a,b] r[n,u-P+a,v-P+b]."""
    d = _c(d, dtype); r = _c(r, dtype)
    N, H, W = r.shape
    K, s, _ = d.shape
    out = np.empty((N, K, H + s - 1, W + s - 1), dtype=dtype)
    getattr(lib(), f"oracle_dtr_{_suf(dtype)}")(N, K, s, H, W, _p(d), _p(r), _p(out))
    return out


def filter_grad(r, z, dtype=np.float64) -> np.ndarray:
    """g[k,a,b] = sum_n sum_ij r[n,i,j] z[n,k,i+P-a,j+P-b] (fp64)."""
    r = _c(r, dtype); z = _c(z, dtype)
    N, K, Hc, Wc = z.shape
    H, W = r.shape[1:]
    s = Hc - H + 1
    g = np.empty((K, s, s), dtype=np.float64)
    getattr(lib(), f"oracle_filter_grad_{_suf(dtype)}")(N, K, s, H, W, _p(r), _p(z), _p(g))
    return g


def lipschitz(d, dtype=np.float32) -> float:
    d = _c(d, dtype)
    K, s, _ = d.shape
    return float(getattr(lib(), f"oracle_lipschitz_{_suf(dtype)}")(K, s, _p(d)))


def code_step(x, d, z, lam, step_z, p, seed, t, dtype=np.float32, rule="lipschitz", mask="entry"):
    """One masked prox-gradient code step.  Returns (z_new, tau_used).

    rule (used when step_z == 0): "lipschitz" -> tau = 1/L_D (reading R8), tau_used a float;
    "eso" -> tau_k = 1/(p L_D + (1-p)||d_k||^2) per filter (E1),
    tau_used an array of K values."""
    x = _c(x, dtype); d = _c(d, dtype)
    z = np.array(z, dtype=dtype, copy=True, order="C")
    N, K, Hc, Wc = z.shape
    s = d.shape[-1]
    H, W = Hc - s + 1, Wc - s + 1
    eso = 1 if (rule == "eso" and not step_z > 0) else 0
    if rule not in ("lipschitz", "eso"):
        raise ValueError(rule)
    tau = np.zeros(max(K, 1), dtype=np.float64)
    getattr(lib(), f"oracle_code_step_{_suf(dtype)}")(
        N, K, s, H, W, _p(x), _p(d), _p(z), float(lam), float(step_z), float(p),
        int(seed) & (2**64 - 1), int(t) & 0xffffffff, _p(tau), eso, MASK_MODES[mask])
    return z, (tau.copy() if eso else float(tau[0]))


ADMM_ITERS = 10      # P:317-318 "the ADMM iteration fixed to 10"
ADMM_ALPHA = 1.8     # P:319-320 over-relaxation
ADMM_CG_ITERS = 5    # reading A3: the paper leaves the CG length to its supplement


def admm_code_step(x, d, z, lam, p, seed, t, rho=None, alpha=ADMM_ALPHA, n_admm=ADMM_ITERS, n_cg=ADMM_CG_ITERS,
                   dtype=np.float32):
    """ADMM masked-LASSO code step, rho = 10 lambda by default
    (P:318-319).  Returns z_new."""
    x = _c(x, dtype); d = _c(d, dtype)
    z = np.array(z, dtype=dtype, copy=True, order="C")
    N, K, Hc, Wc = z.shape
    s = d.shape[-1]
    H, W = Hc - s + 1, Wc - s + 1
    rho = 10.0 * lam if rho is None else rho
    getattr(lib(), f"oracle_admm_code_step_{_suf(dtype)}")(
        N, K, s, H, W, _p(x), _p(d), _p(z), float(lam), float(rho), float(alpha), int(n_admm), int(n_cg),
        float(p), int(seed) & (2**64 - 1), int(t) & 0xffffffff)
    return z


def filter_step(x, d, z, step_d=0.0, dtype=np.float32):
    """One projected-gradient filter step.  Returns (d_new, tau_used, g_fp64, ||Zg||^2)."""
    x = _c(x, dtype); z = _c(z, dtype)
    d = np.array(d, dtype=dtype, copy=True, order="C")
    N, K, Hc, Wc = z.shape
    s = d.shape[-1]
    H, W = Hc - s + 1, Wc - s + 1
    tau = np.zeros(1, dtype=np.float64)
    g = np.zeros((K, s, s), dtype=np.float64)
    zg2 = np.zeros(1, dtype=np.float64)
    getattr(lib(), f"oracle_filter_step_{_suf(dtype)}")(
        N, K, s, H, W, _p(x), _p(d), _p(z), float(step_d), _p(tau), _p(g), _p(zg2))
    return d, float(tau[0]), g, float(zg2[0])


BCD_RIDGE = 1e-10  # reading B2: ridge eps * tr(C_kk) / M in the block solve


def filter_step_bcd(x, d, z, sweeps=1, dtype=np.float32):
    """Projected block-coordinate descent on the filters: per filter
    k in order, the exact minimiser of the Eq.5 quadratic in d_k (others fixed), projected on the unit
    ball.  Returns (d_new, flags) with flags[k] = 1 for a filter left unchanged (no nonzero code)."""
    x = _c(x, dtype); z = _c(z, dtype)
    d = np.array(d, dtype=dtype, copy=True, order="C")
    N, K, Hc, Wc = z.shape
    s = d.shape[-1]
    H, W = Hc - s + 1, Wc - s + 1
    flags = np.zeros(K, dtype=np.uint8)
    getattr(lib(), f"oracle_filter_step_bcd_{_suf(dtype)}")(
        N, K, s, H, W, _p(x), _p(d), _p(z), int(sweeps), _p(flags))
    return d, flags


def surrogate_update(x, z, C, B, t, dtype=np.float32):
    """Eq.7 in place on C [K][K][M][M] and B [K][M] (fp64, block-major): t is the count
    after this mini-batch (t >= 1).  SURVEY.md §8f NEXT-2."""
    x = _c(x, dtype); z = _c(z, dtype)
    N, K, Hc, Wc = z.shape
    s = int(round(np.sqrt(C.shape[-1])))
    H, W = Hc - s + 1, Wc - s + 1
    assert C.dtype == np.float64 and B.dtype == np.float64 and C.flags.c_contiguous and B.flags.c_contiguous
    getattr(lib(), f"oracle_surrogate_update_{_suf(dtype)}")(N, K, s, H, W, _p(x), _p(z), _p(C), _p(B), int(t))


def filter_step_surrogate(C, B, d, sweeps=1, dtype=np.float32):
    """Eq.8: projected block-coordinate sweep(s) on 1/2 d^T C d - d^T B, ||d_k|| <= 1.
    Returns (d_new, flags)."""
    d = np.array(d, dtype=dtype, copy=True, order="C")
    K, s = d.shape[0], d.shape[-1]
    flags = np.zeros(K, dtype=np.uint8)
    getattr(lib(), f"oracle_filter_step_surrogate_{_suf(dtype)}")(K, s, _p(np.ascontiguousarray(C)),
                                                                  _p(np.ascontiguousarray(B)), _p(d),
                                                                  int(sweeps), _p(flags))
    return d, flags


def objective(x, d, z, lam, dtype=np.float32):
    """(F, 1/2||Dz-x||^2, lam*||z||_1) in fp64."""
    x = _c(x, dtype); d = _c(d, dtype); z = _c(z, dtype)
    N, K, Hc, Wc = z.shape
    s = d.shape[-1]
    H, W = Hc - s + 1, Wc - s + 1
    out = np.zeros(3, dtype=np.float64)
    getattr(lib(), f"oracle_objective_{_suf(dtype)}")(N, K, s, H, W, _p(x), _p(d), _p(z), float(lam),
                                                     _p(out))
    return float(out[0]), float(out[1]), float(out[2])


def iteration(x, d, z, lam, p, seed, t, step_z=0.0, step_d=0.0, dtype=np.float32):
    """One SBCSC outer iteration (Alg.1): code step with mask t,
    filter step, then the Eq.1 objective with the new (z, d).  Returns a dict."""
    z1, tau_z = code_step(x, d, z, lam, step_z, p, seed, t, dtype=dtype)
    d1, tau_d, g, zg2 = filter_step(x, d, z1, step_d, dtype=dtype)
    F = objective(x, d1, z1, lam, dtype=dtype)
    return {"z": z1, "d": d1, "tau_z": tau_z, "tau_d": tau_d, "g": g, "zg2": zg2, "F": F}

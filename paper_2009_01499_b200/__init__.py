"""Thin Python binding of libiga2l.so (the C-ABI in include/iga2l.h).

Argument marshalling only: every step of the two-level iteration runs in the library's CUDA
kernels.  Vectors may be CUDA torch tensors (device pointers, used in place on the context
stream) or float64 numpy arrays / CPU tensors (host pointers, staged by the library).
There is no CPU fallback: if the shared library is missing, importing ``lib()`` raises.
"""
import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IGA2L_LIB") or os.path.join(_HERE, "libiga2l.so")   # IGA2L_LIB: A/B builds (dev)
HEADER = os.path.join(os.path.dirname(_HERE), "include", "iga2l.h")

OK, EPARAM, ENUMERIC, NOTCONV, ECUDA, ENCCL, ENOMEM = range(7)
COARSE_EXACT, COARSE_VCYCLE = 0, 1
GEOM_SQUARE, GEOM_QUARTER_ANNULUS = 0, 1


class Opts(ctypes.Structure):
    _fields_ = [("coarse_mode", ctypes.c_int), ("coarse_h_factor", ctypes.c_int),
                ("vcycle_coarsest_m", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("use_graph", ctypes.c_int), ("nranks", ctypes.c_int), ("rank", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p), ("geometry", ctypes.c_int)]


class Info(ctypes.Structure):
    _fields_ = [("n1", ctypes.c_int64), ("N", ctypes.c_int64), ("n1c", ctypes.c_int64),
                ("Nc", ctypes.c_int64), ("colours", ctypes.c_int), ("levels", ctypes.c_int),
                ("launches_per_iter", ctypes.c_int), ("sweep_flops", ctypes.c_double),
                ("iter_hbm_bytes", ctypes.c_double), ("vc_smem_level", ctypes.c_int), ("vc_smem_cs", ctypes.c_int)]


class IgaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"iga2l error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libiga2l.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, i64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    sig = {
        "iga2l_default_opts": (None, [P(Opts)]),
        "iga2l_setup": (i, [i, i, i, i64, i, i, P(vp)]),
        "iga2l_setup_ex": (i, [i, i, i, i64, i, i, P(Opts), P(vp)]),
        "iga2l_sizes": (i, [vp, P(i64), P(i64), P(i64), P(i64)]),
        "iga2l_rhs_sine": (i, [vp, vp]),
        "iga2l_rhs": (i, [vp, vp]),
        "iga2l_apply": (i, [vp, vp, vp]),
        "iga2l_residual_norm": (i, [vp, vp, vp, P(d)]),
        "iga2l_iterate": (i, [vp, vp, vp, i, vp]),
        "iga2l_host_periodic_fd": (i, [i, i, vp, vp]),
        "iga2l_lfa_torus": (i, [i, i, i, i, i, i, i, ctypes.c_ulonglong, vp, vp]),
        "iga2l_solve": (i, [vp, vp, vp, d, i, P(i), P(d)]),
        "iga2l_sweep": (i, [vp, vp, vp, i, i]),
        "iga2l_defect_restrict": (i, [vp, vp, vp, vp]),
        "iga2l_coarse_solve": (i, [vp, vp, vp]),
        "iga2l_prolong_add": (i, [vp, vp, vp]),
        "iga2l_get_info": (i, [vp, P(Info)]),
        "iga2l_host_band_tables": (i, [i, i64, vp, vp]),
        "iga2l_host_coarse_fd": (i, [i, i64, vp, vp]),
        "iga2l_host_restriction_1d": (i, [i, i, i64, i, vp]),
        "iga2l_host_slab_plan": (i, [i, i, i, i64, i, i, vp]),
        "iga2l_host_annulus_tables": (i, [i, i64, vp, vp]),
        "iga2l_host_annulus_restriction_1d": (i, [i, i, i, i64, i, vp]),
        "iga2l_host_annulus_load": (i, [i, i64, vp]),
        "iga2l_nccl_unique_id": (i, [vp]),
        "iga2l_destroy": (i, [vp]),
        "iga2l_last_error": (ctypes.c_char_p, []),
        "iga2l_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def header_symbols():
    """Every function the public header declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(iga2l_[a-z0-9_]+)\s*\(", txt)))


def _check(rc, allow=()):
    if rc != OK and rc not in allow:
        raise IgaError(rc, lib().iga2l_last_error().decode())
    return rc


def _ptr(a):
    """Pointer of a float64 contiguous torch tensor (device or host) or numpy array."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError("vectors must be contiguous float64")
        return ctypes.c_void_p(a.data_ptr())
    import numpy as np
    if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        raise TypeError("vectors must be C-contiguous float64")
    return ctypes.c_void_p(a.ctypes.data)


def host_band_tables(p, m):
    import numpy as np
    n1 = m + p - 2
    K = np.zeros(n1 * (2 * p + 1))
    M = np.zeros_like(K)
    _check(lib().iga2l_host_band_tables(p, m, _ptr(K), _ptr(M)))
    return K.reshape(n1, 2 * p + 1), M.reshape(n1, 2 * p + 1)


def host_coarse_fd(q, m):
    """1D generalised eigen-decomposition of the degree-q level (host-only): V (n x n), lam (n)."""
    import numpy as np
    n = m + q - 2
    V = np.zeros(n * n)
    lam = np.zeros(n)
    _check(lib().iga2l_host_coarse_fd(q, m, _ptr(V), _ptr(lam)))
    return V.reshape(n, n), lam


def host_periodic_fd(q, n):
    """1D generalised eigen-decomposition of the degree-q level on the n-point torus (host-only)."""
    import numpy as np
    V = np.zeros(n * n)
    lam = np.zeros(n)
    _check(lib().iga2l_host_periodic_fd(q, n, _ptr(V), _ptr(lam)))
    return V.reshape(n, n), lam


def host_slab_plan(dim, p, block, m, nranks, rank):
    """Slab plan (z0, z1, za, zb, centre_lo, centre_hi, H, feasible) of `rank` (host-only)."""
    import numpy as np
    out = np.zeros(8, dtype=np.int64)
    _check(lib().iga2l_host_slab_plan(dim, p, block, m, nranks, rank, ctypes.c_void_p(out.ctypes.data)))
    return dict(zip(["z0", "z1", "za", "zb", "c_lo", "c_hi", "H", "feasible"], [int(v) for v in out]))


def nccl_unique_id():
    buf = (ctypes.c_char * 128)()
    _check(lib().iga2l_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


def host_restriction_1d(p, q, m, h_factor):
    import numpy as np
    n1 = m + p - 2
    n1c = m // h_factor + q - 2
    R = np.zeros(n1c * n1)
    _check(lib().iga2l_host_restriction_1d(p, q, m, h_factor, _ptr(R)))
    return R.reshape(n1c, n1)


def host_annulus_tables(p, m):
    """Quarter-annulus per-axis band tables (host-only): (Kx, Mx, Ky, My), each (n1, 2p+1)."""
    import numpy as np
    n1 = m + p - 2
    K = np.zeros(2 * n1 * (2 * p + 1))
    M = np.zeros_like(K)
    _check(lib().iga2l_host_annulus_tables(p, m, _ptr(K), _ptr(M)))
    K, M = K.reshape(2, n1, 2 * p + 1), M.reshape(2, n1, 2 * p + 1)
    return K[0], M[0], K[1], M[1]


def host_annulus_restriction_1d(axis, p, q, m, h_factor):
    import numpy as np
    n1, n1c = m + p - 2, m // h_factor + q - 2
    R = np.zeros(n1c * n1)
    _check(lib().iga2l_host_annulus_restriction_1d(axis, p, q, m, h_factor, _ptr(R)))
    return R.reshape(n1c, n1)


def host_annulus_load(p, m):
    import numpy as np
    b = np.zeros((m + p - 2) ** 2)
    _check(lib().iga2l_host_annulus_load(p, m, _ptr(b)))
    return b


def lfa_torus(p, q, n, block, h_factor=1, iters=200, seed=0, dim=2, return_ratios=False):
    """iga2l_lfa_torus: spectral radius of the two-grid error operator on the n x n torus (power iteration
    with the library's kernels; see the header)."""
    rho = ctypes.c_double()
    rat = (ctypes.c_double * iters)()
    _check(lib().iga2l_lfa_torus(dim, p, q, n, block, h_factor, iters, seed, ctypes.byref(rho),
                                 ctypes.cast(rat, ctypes.c_void_p)))
    return (rho.value, list(rat)) if return_ratios else rho.value


class Context:
    """One iga2l context (iga2l_setup_ex).  Methods mirror the C entry points."""

    def __init__(self, dim, p, q, m, block, overlap=None, coarse_mode=COARSE_VCYCLE, coarse_h_factor=2,
                 vcycle_coarsest_m=8, stream=None, use_graph=True, nranks=1, rank=0, nccl_id=None,
                 geometry="square"):
        L = lib()
        o = Opts()
        L.iga2l_default_opts(ctypes.byref(o))
        o.coarse_mode, o.coarse_h_factor, o.vcycle_coarsest_m = coarse_mode, coarse_h_factor, vcycle_coarsest_m
        o.use_graph = int(bool(use_graph))
        if stream is None:          # default: torch's current stream (0 = legacy -> library's own blocking stream)
            try:
                import torch
                stream = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
            except Exception:
                stream = None
        o.stream = stream or None
        o.nranks, o.rank = nranks, rank
        o.geometry = {"square": GEOM_SQUARE, "annulus": GEOM_QUARTER_ANNULUS}[geometry]
        self._id = None
        if nccl_id is not None:
            self._id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._id, ctypes.c_void_p)
        self._h = ctypes.c_void_p()
        ov = block - 1 if overlap is None else overlap
        _check(L.iga2l_setup_ex(dim, p, q, m, block, ov, ctypes.byref(o), ctypes.byref(self._h)))
        self.dim, self.p, self.q, self.m, self.s = dim, p, q, m, block
        info = self.info()
        self.n1, self.N, self.n1c, self.Nc = info.n1, info.N, info.n1c, info.Nc
        nl, z0, z1 = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(L.iga2l_sizes(self._h, ctypes.byref(nl), ctypes.byref(z0), ctypes.byref(z1), None))
        self.N_local, self.z0, self.z1 = nl.value, z0.value, z1.value

    def info(self):
        inf = Info()
        _check(lib().iga2l_get_info(self._h, ctypes.byref(inf)))
        return inf

    def rhs(self, b):
        """The paper's right-hand side for this geometry (square: sine; annulus: P:439-447)."""
        _check(lib().iga2l_rhs(self._h, _ptr(b)))
        return b

    def rhs_sine(self, b):
        _check(lib().iga2l_rhs_sine(self._h, _ptr(b)))
        return b

    def apply(self, x, y):
        _check(lib().iga2l_apply(self._h, _ptr(x), _ptr(y)))
        return y

    def residual_norm(self, b, x):
        out = ctypes.c_double()
        _check(lib().iga2l_residual_norm(self._h, _ptr(b), _ptr(x), ctypes.byref(out)))
        return out.value

    def iterate(self, b, x, iters=1, res_hist=None):
        _check(lib().iga2l_iterate(self._h, _ptr(b), _ptr(x), iters, _ptr(res_hist)))
        return x

    def solve(self, b, x, rtol=1e-8, maxit=100):
        it, rr = ctypes.c_int(), ctypes.c_double()
        rc = _check(lib().iga2l_solve(self._h, _ptr(b), _ptr(x), rtol, maxit, ctypes.byref(it), ctypes.byref(rr)),
                    allow=(NOTCONV,))
        return it.value, rr.value, rc == OK

    def sweep(self, b, x, colour_begin=0, colour_end=None):
        ce = self.info().colours if colour_end is None else colour_end
        _check(lib().iga2l_sweep(self._h, _ptr(b), _ptr(x), colour_begin, ce))
        return x

    def defect_restrict(self, b, x, dq):
        _check(lib().iga2l_defect_restrict(self._h, _ptr(b), _ptr(x), _ptr(dq)))
        return dq

    def coarse_solve(self, dq, e):
        _check(lib().iga2l_coarse_solve(self._h, _ptr(dq), _ptr(e)))
        return e

    def prolong_add(self, e, x):
        _check(lib().iga2l_prolong_add(self._h, _ptr(e), _ptr(x)))
        return x

    def close(self):
        if self._h:
            lib().iga2l_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""Thin ctypes binding of libxc.so (include/xc.h): argument marshalling only.

Every step of the transform runs in the library's sm_100a kernels; PyTorch is
used for device memory and streams.  There is no CPU fallback: if libxc.so is
missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libxc.so")

XC_COS, XC_JACOBI, XC_LAGUERRE, XC_EXP, XC_LAGSPEC, XC_LAG2D = 1, 2, 3, 4, 5, 6
COMPLEX_KINDS = (XC_EXP, XC_LAGSPEC)  # planar complex X / Y (real rows, then imaginary rows)
XC_DIR_A, XC_DIR_WAT = 1, 2
_STATUS = {0: "XC_OK", 1: "XC_EINVAL", 2: "XC_ENUMERIC", 3: "XC_ESTATE", 4: "XC_ENOMEM", 5: "XC_ECUDA",
           6: "XC_EUNSUPPORTED", 7: "XC_ENCCL"}

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)


class XcParams(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("eps1", ctypes.c_double),
                ("eps2", ctypes.c_double), ("dense_cutoff", ctypes.c_int), ("dirs", ctypes.c_int),
                ("weights", _dp), ("device", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("node_chunk", ctypes.c_int), ("eta", ctypes.c_double), ("n_rows", _i64),
                ("trig_precompute", ctypes.c_int), ("thresh_mode", ctypes.c_int),
                ("apply_path", ctypes.c_int)]


class XcInfo(ctypes.Structure):
    _fields_ = [("N", _i64), ("kind", ctypes.c_int), ("zeta", ctypes.c_double), ("eps1", ctypes.c_double),
                ("eps2", ctypes.c_double), ("n_blocks", ctypes.c_int), ("tail", ctypes.c_int),
                ("dirs", ctypes.c_int), ("nnz", _i64), ("op_bytes_A", _i64), ("op_bytes_WAT", _i64),
                ("flops_per_col_A", ctypes.c_double), ("flops_per_col_WAT", ctypes.c_double),
                ("dmma_flops_per_col_A", ctypes.c_double), ("dmma_flops_per_col_WAT", ctypes.c_double),
                ("launches_A", ctypes.c_int), ("launches_WAT", ctypes.c_int), ("M", _i64),
                ("alg_bytes_per_col", ctypes.c_double), ("alg_bytes_fixed", ctypes.c_double)]


class XcExchange(ctypes.Structure):
    _fields_ = [("send", ctypes.c_void_p), ("recv", ctypes.c_void_p), ("bytes_per_rank", ctypes.c_size_t)]


class XcBlockInfo(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("H", ctypes.c_int), ("m_off", ctypes.c_int), ("keep_lo", ctypes.c_int),
                ("keep_hi", ctypes.c_int), ("nnz", _i64), ("max_band", ctypes.c_int), ("q_taps", ctypes.c_int)]


EXPORTS = ["xc_params_default", "xc_build_compressed", "xc_build_from_bands", "xc_build_local", "xc_build_step", "xc_apply", "xc_c2r_check", "xc_set_graphs", "xc_apply_host", "xc_apply_host_async", "xc_host_wait", "xc_reserve",
           "xc_attach_workspace", "xc_launches", "xc_export", "xc_import",
           "xc_debug_guards",
           "xc_workspace_query", "xc_info", "xc_block_info", "xc_block_window", "xc_node_spectrum",
           "xc_gauss_rule", "xc_plan_chain", "xc_profile_enable", "xc_profile_read", "xc_destroy",
           "xc_last_error", "xc_version"]

_lib = None


class XcError(RuntimeError):
    pass


def load():
    """Load libxc.so (built by __graft_entry__.build() / `make -C paper_2004_11610_b200/csrc`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise XcError(f"libxc.so not built ({LIB_PATH}); run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    lib.xc_params_default.argtypes = [ctypes.POINTER(XcParams)]
    lib.xc_build_compressed.argtypes = [ctypes.c_int, ctypes.POINTER(XcParams), _dp, _i64, ctypes.c_double,
                                        ctypes.POINTER(vp)]
    lib.xc_build_local.argtypes = [ctypes.c_int, ctypes.POINTER(XcParams), _dp, _i64, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(XcExchange)]
    lib.xc_build_step.argtypes = [vp, ctypes.POINTER(XcExchange)]
    lib.xc_build_from_bands.argtypes = [ctypes.c_int, ctypes.POINTER(XcParams), _dp, _i64, ctypes.c_double,
                                        ctypes.POINTER(ctypes.POINTER(ctypes.c_int)),
                                        ctypes.POINTER(ctypes.POINTER(ctypes.c_int)), ctypes.POINTER(_dp),
                                        ctypes.POINTER(vp)]
    lib.xc_apply.argtypes = [vp, ctypes.c_int, vp, _i64, vp, _i64, _i64, vp]
    lib.xc_apply_host.argtypes = [vp, ctypes.c_int, vp, vp, _i64, vp]
    lib.xc_set_graphs.argtypes = [vp, ctypes.c_int]
    lib.xc_c2r_check.argtypes = [_i64, vp, _i64, vp, _i64, _i64, vp]
    lib.xc_apply_host_async.argtypes = [vp, ctypes.c_int, vp, vp, _i64, vp]
    lib.xc_host_wait.argtypes = [vp]
    lib.xc_reserve.argtypes = [vp, _i64]
    lib.xc_attach_workspace.argtypes = [vp, vp, vp, ctypes.c_size_t]
    lib.xc_launches.argtypes = [vp, ctypes.c_int, _i64, ctypes.POINTER(_i64)]
    lib.xc_export.argtypes = [vp, ctypes.c_char_p]
    lib.xc_debug_guards.argtypes = [vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
    lib.xc_import.argtypes = [ctypes.c_char_p, ctypes.POINTER(XcParams), ctypes.POINTER(vp)]
    lib.xc_workspace_query.argtypes = [vp, _i64, ctypes.POINTER(ctypes.c_size_t)]
    lib.xc_info.argtypes = [vp, ctypes.POINTER(XcInfo)]
    lib.xc_block_info.argtypes = [vp, ctypes.c_int, ctypes.POINTER(XcBlockInfo)]
    lib.xc_block_window.argtypes = [vp, ctypes.c_int, _dp]
    lib.xc_node_spectrum.argtypes = [vp, ctypes.c_int, _i64, _dp, _dp]
    lib.xc_gauss_rule.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _i64, _dp, _dp, _dp,
                                  ctypes.c_int]
    ip = ctypes.POINTER(ctypes.c_int)
    lib.xc_plan_chain.argtypes = [ctypes.c_int, _i64, ctypes.c_double, ctypes.c_double, ctypes.c_int, _dp, ip,
                                  ip, ip, ip, ip, ctypes.c_int, ip]
    lib.xc_profile_enable.argtypes = [vp, ctypes.c_int]
    lib.xc_profile_read.argtypes = [vp, _dp, _dp, _dp, _dp, ctypes.POINTER(_i64)]
    lib.xc_destroy.argtypes = [vp]
    lib.xc_destroy.restype = None
    lib.xc_last_error.restype = ctypes.c_char_p
    lib.xc_version.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("xc_destroy", "xc_last_error", "xc_version"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(rc: int):
    if rc != 0:
        msg = load().xc_last_error().decode(errors="replace")
        raise XcError(f"{_STATUS.get(rc, rc)}: {msg}")


def _np_ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def gauss_rule(kind: int, N: int, alpha: float = 0.0, beta: float = 0.0, device: int = 0):
    """Gauss nodes (ascending), weights and wt (= w e^x for Laguerre) computed on the GPU."""
    lib = load()
    x = np.empty(N)
    w = np.empty(N)
    wt = np.empty(N)
    _check(lib.xc_gauss_rule(kind, alpha, beta, N, _np_ptr(x), _np_ptr(w), _np_ptr(wt), device))
    return x, w, wt


def plan_chain(kind: int, N: int, eps1: float, eps2: float = 0.0, dense_cutoff: int = 0):
    """Host-only planning: (zeta, [(L, m_off, keep_lo, keep_hi)], tail)."""
    lib = load()
    M = 64
    z = ctypes.c_double()
    nb, tail = ctypes.c_int(), ctypes.c_int()
    arrs = [(ctypes.c_int * M)() for _ in range(4)]
    _check(lib.xc_plan_chain(kind, N, eps1, eps2, dense_cutoff, ctypes.byref(z), ctypes.byref(nb), *arrs, M,
                             ctypes.byref(tail)))
    blocks = [tuple(a[i] for a in arrs) for i in range(nb.value)]
    return z.value, blocks, tail.value


def device_bytes(ptr: int, nbytes: int, device: int = 0):
    """A uint8 CUDA tensor viewing `nbytes` of library-owned device memory (no copy)."""
    import torch

    class _View:
        pass

    v = _View()
    v.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                  "strides": None}
    return torch.as_tensor(v, device=f"cuda:{device}")


def nccl_allgather(group=None):
    """The exchange of a distributed build as one torch.distributed all-gather (NCCL on GPUs):
    recv[r * n : (r + 1) * n] = send of rank r."""
    import torch.distributed as dist

    def ag(send, recv):
        dist.all_gather_into_tensor(recv, send, group=group)
    return ag


def host_allgather(group=None):
    """The same exchange through host memory (a gloo process group): device send -> host, all-gather,
    host -> device recv.  For process groups without a GPU transport (tests of two processes on
    one GPU; no kernel waits on another process, the exchange is host-mediated)."""
    import torch
    import torch.distributed as dist

    def ag(send, recv):
        h = send.cpu()
        parts = [torch.empty_like(h) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, h, group=group)
        recv.copy_(torch.cat(parts).to(recv.device))
    return ag


class Transform:
    """A compressed special-function transform (handle of xc_build_compressed).

    dist=(rank, nranks, allgather): distributed precompute -- this rank computes
    the node bands of its node range, `allgather(send, recv)` (uint8 CUDA tensors, recv
    rank-major; e.g. nccl_allgather()) exchanges them, and every rank ends with the whole
    operator (identical to the single-process build)."""

    def __init__(self, kind: int, nodes, eps: float, alpha: float = 0.0, beta: float = 0.0,
                 eps1: float = 0.0, eps2: float = 0.0, dense_cutoff: int = 0, dirs: int = XC_DIR_A,
                 weights=None, device: int = 0, node_chunk: int = 0, stream=None, dist=None,
                 eta: float = 0.0, n_rows: int = 0, trig_precompute: int = 0, thresh_mode: int = 0,
                 apply_path: int = 0):
        lib = load()
        self._lib = lib
        self.kind = kind
        self._reserved, self._attached = 0, {}
        x = np.ascontiguousarray(np.asarray(nodes, dtype=np.float64))
        self.N = x.size
        self.M = n_rows if n_rows > 0 else self.N   # degrees (rows of A)
        p = XcParams()
        lib.xc_params_default(ctypes.byref(p))
        p.alpha, p.beta, p.eps1, p.eps2 = alpha, beta, eps1, eps2
        p.dense_cutoff, p.dirs, p.device, p.node_chunk = dense_cutoff, dirs, device, node_chunk
        p.eta, p.n_rows, p.trig_precompute, p.thresh_mode = eta, n_rows, trig_precompute, thresh_mode
        p.apply_path = apply_path
        self._w = None
        if weights is not None:
            self._w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
            p.weights = _np_ptr(self._w)
        p.stream = ctypes.c_void_p(stream) if stream else None
        h = ctypes.c_void_p()
        self.device = device
        if dist is None:
            _check(lib.xc_build_compressed(kind, ctypes.byref(p), _np_ptr(x), self.N, eps, ctypes.byref(h)))
            self._h = h
            return
        import torch
        rank, nranks, allgather = dist
        ex = XcExchange()
        _check(lib.xc_build_local(kind, ctypes.byref(p), _np_ptr(x), self.N, eps, rank, nranks, ctypes.byref(h),
                                  ctypes.byref(ex)))
        self._h = h
        self.exchanges = []
        while ex.bytes_per_rank:
            n = ex.bytes_per_rank
            send = device_bytes(ex.send, n, device)
            recv = device_bytes(ex.recv, n * nranks, device)
            torch.cuda.synchronize(device)
            try:
                allgather(send, recv)
                torch.cuda.synchronize(device)
            except Exception as e:   # the exchange failed (NCCL / process group error)
                lib.xc_destroy(self._h)
                self._h = None
                raise XcError(f"XC_ENCCL: exchange all-gather failed: {e}") from e
            self.exchanges.append(n)
            _check(lib.xc_build_step(self._h, ctypes.byref(ex)))

    @classmethod
    def from_bands(cls, kind: int, nodes, eps: float, bands, **kw):
        """xc_build_from_bands: the computation stage on caller-supplied node bands, one
        (start int32[N], len int32[N], vals complex128[sum len]) triple per block of the plan."""
        lib = load()
        self = cls.__new__(cls)
        self._lib = lib
        self.kind = kind
        self._reserved, self._attached = 0, {}
        x = np.ascontiguousarray(np.asarray(nodes, dtype=np.float64))
        self.N = x.size
        self.M = kw.get("n_rows", 0) or self.N
        p = XcParams()
        lib.xc_params_default(ctypes.byref(p))
        for k, v in kw.items():
            if k == "weights":
                self._w = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
                p.weights = _np_ptr(self._w)
            else:
                setattr(p, k, v)
        nb = len(bands)
        keep = []
        st = (ctypes.POINTER(ctypes.c_int) * nb)()
        ln = (ctypes.POINTER(ctypes.c_int) * nb)()
        vl = (_dp * nb)()
        for i, (s0, l0, v0) in enumerate(bands):
            s0 = np.ascontiguousarray(s0, dtype=np.int32)
            l0 = np.ascontiguousarray(l0, dtype=np.int32)
            v0 = np.ascontiguousarray(np.asarray(v0, dtype=np.complex128)).view(np.float64)
            keep += [s0, l0, v0]
            st[i] = s0.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
            ln[i] = l0.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
            vl[i] = _np_ptr(v0) if v0.size else _np_ptr(np.zeros(2))
        h = ctypes.c_void_p()
        self.device = kw.get("device", 0)
        _check(lib.xc_build_from_bands(kind, ctypes.byref(p), _np_ptr(x), self.N, eps, st, ln, vl, ctypes.byref(h)))
        self._h = h
        return self

    @classmethod
    def load_file(cls, path: str, device: int = 0):
        """xc_import: the operator of an xc_export file (plan recomputed and checked, kept values
        from the file: applies bit-identical to the exporting handle's)."""
        lib = load()
        self = cls.__new__(cls)
        self._lib = lib
        self._reserved, self._attached = 0, {}
        p = XcParams()
        lib.xc_params_default(ctypes.byref(p))
        p.device = device
        h = ctypes.c_void_p()
        _check(lib.xc_import(os.fsencode(path), ctypes.byref(p), ctypes.byref(h)))
        self._h = h
        self.device = device
        inf = self.info()
        self.kind, self.N, self.M = inf["kind"], inf["N"], inf["M"]
        return self

    def export(self, path: str):
        """xc_export: write the compressed operator to `path` (versioned file, include/xc.h)."""
        _check(self._lib.xc_export(self._h, os.fsencode(path)))

    # -- computation stage --------------------------------------------------------------
    def apply(self, X, direction: int = XC_DIR_A, out=None, stream=None):
        """Y = A X (XC_DIR_A) or diag(wt) A^T X (XC_DIR_WAT); X a CUDA fp64 tensor (N x B)."""
        import torch
        # argument checks only (cheap attribute reads: for the microsecond-scale configs the
        # binding's own cost is part of every call)
        if not (isinstance(X, torch.Tensor) and X.is_cuda and X.dtype == torch.float64 and X.dim() == 2):
            raise XcError("X must be a 2-D CUDA float64 tensor")
        if X.stride(1) != 1:
            X = X.contiguous()
        N, B = X.shape
        rin, rout = self.rows(direction)
        if N != rin:
            raise XcError(f"X has {N} rows, transform needs {rin}")
        dev = X.get_device()
        if out is None:
            out = torch.empty((rout, B), dtype=torch.float64, device=X.device)
        elif not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float64 and out.dim() == 2
                  and out.shape[0] == rout and out.shape[1] == B and out.get_device() == dev
                  and out.stride(1) == 1 and out.stride(0) >= B):
            raise XcError(f"out must be a CUDA float64 tensor of shape ({rout}, {B}) on {X.device} with "
                          f"unit column stride")
        st = stream if stream is not None else torch._C._cuda_getCurrentRawStream(dev)
        if B > self._reserved and st not in self._attached:   # xc_apply itself never allocates
            self.reserve(B)
        rc = self._lib.xc_apply(self._h, direction, X.data_ptr(), X.stride(0), out.data_ptr(), out.stride(0), B, st)
        if rc:
            _check(rc)
        return out

    def rows(self, direction: int = XC_DIR_A):
        """(rows of X, rows of Y) of an apply: nodes N / degrees M by direction, twice for the
        planar complex kinds."""
        r = self.__dict__.get("_rows_cache")
        if r is None or r[0] != (self.kind, self.N, self.M):
            cf = 2 if self.kind in COMPLEX_KINDS else 1
            r = ((self.kind, self.N, self.M), (cf * self.N, cf * self.M), (cf * self.M, cf * self.N))
            self._rows_cache = r
        return r[1] if direction == XC_DIR_A else r[2]

    def apply_complex(self, Xc, direction: int = XC_DIR_A, stream=None):
        """Complex kinds with a complex128 CUDA tensor: marshalled to and from the planar layout
        of the C ABI (real rows, then imaginary rows)."""
        import torch
        Xp = torch.cat([Xc.real, Xc.imag]).contiguous()
        Yp = self.apply(Xp, direction, stream=stream)
        h = Yp.shape[0] // 2
        return torch.complex(Yp[:h], Yp[h:])

    def apply_host(self, X: np.ndarray, direction: int = XC_DIR_A, out: np.ndarray | None = None, stream=None):
        """End-to-end call with host buffers (copies inside the library call)."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        N, B = X.shape
        rin, rout = self.rows(direction)
        if N != rin:
            raise XcError(f"X has {N} rows, transform needs {rin}")
        if out is None:
            out = np.empty((rout, B), dtype=np.float64)
        _check(self._lib.xc_apply_host(self._h, direction, ctypes.c_void_p(X.ctypes.data),
                                       ctypes.c_void_p(out.ctypes.data), B, ctypes.c_void_p(stream or 0)))
        return out

    def apply_host_ptr(self, x_ptr: int, y_ptr: int, B: int, direction: int = XC_DIR_A, stream=None):
        _check(self._lib.xc_apply_host(self._h, direction, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr), B,
                                       ctypes.c_void_p(stream or 0)))

    def graphs(self, enable: bool = True):
        """CUDA-graph replay of repeated applies with the same arguments (default on)."""
        _check(self._lib.xc_set_graphs(self._h, 1 if enable else 0))

    def apply_host_async_ptr(self, x_ptr: int, y_ptr: int, B: int, direction: int = XC_DIR_A, stream=None):
        """Streaming host-buffer apply (no wait); see host_wait()."""
        _check(self._lib.xc_apply_host_async(self._h, direction, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr), B,
                                             ctypes.c_void_p(stream or 0)))

    def host_wait(self):
        _check(self._lib.xc_host_wait(self._h))

    def profile(self, enable: bool = True):
        _check(self._lib.xc_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        v = [ctypes.c_double() for _ in range(4)]
        n = _i64()
        _check(self._lib.xc_profile_read(self._h, *[ctypes.byref(a) for a in v], ctypes.byref(n)))
        return {"ms_spmm": v[0].value, "ms_fft": v[1].value, "ms_reduce": v[2].value, "ms_total": v[3].value,
                "n": n.value}

    def reserve(self, B: int):
        """xc_reserve: the handle's own workspace for up to B columns (allocates)."""
        _check(self._lib.xc_reserve(self._h, B))
        self._reserved = max(self._reserved, B)

    def attach_workspace(self, stream: int, ws=None):
        """xc_attach_workspace: bind a caller-owned CUDA tensor (>= workspace_bytes(B) bytes) as the
        workspace of applies on `stream` (a cudaStream_t handle); ws=None detaches."""
        if ws is None:
            _check(self._lib.xc_attach_workspace(self._h, ctypes.c_void_p(stream), None, 0))
            self._attached.pop(stream, None)
            return
        nbytes = ws.numel() * ws.element_size()
        _check(self._lib.xc_attach_workspace(self._h, ctypes.c_void_p(stream), ctypes.c_void_p(ws.data_ptr()),
                                             nbytes))
        self._attached[stream] = ws   # keep the memory alive while attached

    def debug_guards(self):
        """xc_debug_guards: (overwritten guard bytes, guard bytes checked); needs XC_WS_GUARD=1."""
        bad, chk = _i64(), _i64()
        _check(self._lib.xc_debug_guards(self._h, ctypes.byref(bad), ctypes.byref(chk)))
        return bad.value, chk.value

    def launches(self, B: int, direction: int = XC_DIR_A) -> int:
        """Kernel launches one xc_apply of B columns makes (xc_launches)."""
        n = _i64()
        _check(self._lib.xc_launches(self._h, direction, B, ctypes.byref(n)))
        return n.value

    def workspace_bytes(self, B: int) -> int:
        n = ctypes.c_size_t()
        _check(self._lib.xc_workspace_query(self._h, B, ctypes.byref(n)))
        return n.value

    # -- introspection --------------------------------------------------------------------
    def info(self) -> dict:
        s = XcInfo()
        _check(self._lib.xc_info(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in XcInfo._fields_}

    def block_info(self, i: int) -> dict:
        s = XcBlockInfo()
        _check(self._lib.xc_block_info(self._h, i, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in XcBlockInfo._fields_}

    def blocks(self) -> list:
        return [self.block_info(i) for i in range(self.info()["n_blocks"])]

    def window(self, i: int) -> np.ndarray:
        L = self.block_info(i)["L"]
        w = np.empty(L)
        _check(self._lib.xc_block_window(self._h, i, _np_ptr(w)))
        return w

    def node_spectrum(self, i: int, k: int) -> np.ndarray:
        H = self.block_info(i)["H"]
        re, im = np.empty(H), np.empty(H)
        _check(self._lib.xc_node_spectrum(self._h, i, k, _np_ptr(re), _np_ptr(im)))
        return re + 1j * im

    def close(self):
        if getattr(self, "_h", None):
            self._lib.xc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def c2r_check(L: int, U, stream=None):
    """Test entry point: the real-output inverse DFT engine alone (xc_c2r_check); U a complex128
    CUDA tensor (L/2 + 1, B), returns the (L, B) float64 unitary inverse."""
    import torch
    Ui = torch.view_as_real(U.contiguous()).contiguous()
    B = U.shape[1]
    Y = torch.empty((L, B), dtype=torch.float64, device=U.device)
    st = stream if stream is not None else torch.cuda.current_stream(U.device).cuda_stream
    _check(load().xc_c2r_check(L, ctypes.c_void_p(Ui.data_ptr()), B, ctypes.c_void_p(Y.data_ptr()), B, B,
                               ctypes.c_void_p(st)))
    return Y


def version() -> str:
    return load().xc_version().decode()

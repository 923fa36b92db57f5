"""Thin Python binding of libgbla (include/gbla.h) -- argument marshalling only.

Every step of the reduction runs in the CUDA kernels of ``csrc/``.  PyTorch
is used for device memory (the library allocates through torch's caching
allocator via ``gbla_ctx_set_allocator``), streams and process groups.
There is no CPU fallback: importing this package without the built
``libgbla.so`` raises, and every call raises on a non-OK status.

Names follow the C ABI: gbla_splice, gbla_reduce_B, gbla_reduce_C,
gbla_update_D, gbla_echelon_D, gbla_reduce.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgbla.so")

# flags (include/gbla.h)
GBLA_ORDER_NEW = 0x00
GBLA_ORDER_STANDARD = 0x01
GBLA_FUSE_D = 0x02
GBLA_HOST_INPUT = 0x04
GBLA_KEEP_CPRIME = 0x08
GBLA_SPARSE_INT = 0x10
GBLA_DENSE_INT = 0x20
GBLA_DENSE_TC = 0x40
GBLA_ECHELON_REF = 0x80     # echelon_D: row echelon form only

_STATUS = {0: "GBLA_OK", 1: "GBLA_E_INVAL", 2: "GBLA_E_DOMAIN", 3: "GBLA_E_ORDER", 4: "GBLA_E_NOMEM",
           5: "GBLA_E_CUDA", 6: "GBLA_E_NCCL", 7: "GBLA_E_INTERNAL"}


class GblaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class _CSR(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class _FileInfo(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("typecode", ctypes.c_uint32), ("version", ctypes.c_uint32),
                ("p", ctypes.c_uint32), ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("k", ctypes.c_int64), ("pnb", ctypes.c_int64), ("pnnz", ctypes.c_int64)]


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
_MEMQ_FN = ctypes.CFUNCTYPE(ctypes.c_size_t, ctypes.c_void_p)

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libgbla.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libgbla.so not found at {path}: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i64, u32, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int
    P = ctypes.POINTER
    sig = {
        "gbla_ctx_create": ([ctypes.c_int, P(vp)], st),
        "gbla_ctx_set_allocator": ([vp, _ALLOC_FN, _FREE_FN, vp], st),
        "gbla_ctx_set_mem_query": ([vp, _MEMQ_FN, vp], st),
        "gbla_ctx_set_comm": ([vp, vp, ctypes.c_int, ctypes.c_int], st),
        "gbla_ctx_destroy": ([vp], None),
        "gbla_splice": ([vp, P(_CSR), u32, u32, vp, P(vp)], st),
        "gbla_reduce_B": ([vp, vp], st),
        "gbla_reduce_C": ([vp, u32, vp], st),
        "gbla_update_D": ([vp, vp], st),
        "gbla_echelon_D": ([vp, u32, vp, P(i64)], st),
        "gbla_reduce": ([vp, P(_CSR), u32, u32, vp, P(vp)], st),
        "gbla_get_dims": ([vp, P(i64), P(i64), P(i64)], st),
        "gbla_get_maps": ([vp, P(vp), P(vp), P(vp)], st),
        "gbla_get_D": ([vp, P(vp), P(i64)], st),
        "gbla_get_Cprime": ([vp, P(vp), P(i64)], st),
        "gbla_get_Bprime": ([vp, P(vp), P(i64)], st),
        "gbla_densify_quadrant": ([vp, ctypes.c_char, vp, i64, vp], st),
        "gbla_get_rref": ([vp, P(i64), P(vp), P(vp), P(i64)], st),
        "gbla_copy_rref_to_host": ([vp, vp, vp, vp], st),
        "gbla_get_opcount": ([vp, P(ctypes.c_uint64), P(ctypes.c_uint64)], st),
        "gbla_get_phase_ms": ([vp, P(ctypes.c_float)], st),
        "gbla_sync": ([vp], st),
        "gbla_mat_free": ([vp], None),
        "gbla_last_error": ([], ctypes.c_char_p),
        "gbla_version": ([], ctypes.c_char_p),
        "gbla_nccl_get_unique_id": ([vp], st),
        "gbla_kernel_launches": ([], ctypes.c_uint64),
        "gbla_modgemm": ([vp, u32, i64, i64, i64, vp, i64, vp, i64, vp, vp, i64, ctypes.c_int, vp], st),
        "gbla_get_kernel_ms": ([vp, ctypes.c_int, P(ctypes.c_float), P(i64)], st),
        "gbla_get_multilines": ([vp, vp, P(i64), P(vp), P(vp), P(vp)], st),
        "gbla_get_kernel_work": ([vp, ctypes.c_int, P(ctypes.c_uint64)], st),
        "gbla_get_kernel_exec": ([vp, ctypes.c_int, P(ctypes.c_uint64)], st),
        "gbla_modgemm_bench": ([vp, u32, i64, i64, i64, ctypes.c_int, vp, P(ctypes.c_float)], st),
        "gbla_rref_M": ([vp, vp, P(i64)], st),
        "gbla_get_multiline_runs": ([vp, vp, P(i64), P(vp), P(vp), P(vp), P(vp)], st),
        "gbla_reduce_wide": ([vp, P(_CSR), u32, u32, vp, P(vp)], st),
        "gbla_get_wide": ([vp, P(i64), P(vp), P(vp), P(vp), P(i64)], st),
        "gbla_file_info_parse": ([vp, ctypes.c_size_t, ctypes.c_int, P(_FileInfo)], st),
        "gbla_file_decode": ([vp, vp, ctypes.c_size_t, ctypes.c_int, vp, vp, vp, vp], st),
        "gbla_get_rref_M": ([vp, P(_CSR)], st),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def exported_symbols():
    """Names the binding expects the library to export (tests check them)."""
    return ["gbla_ctx_create", "gbla_ctx_set_allocator", "gbla_ctx_set_mem_query", "gbla_ctx_set_comm",
            "gbla_ctx_destroy",
            "gbla_splice", "gbla_reduce_B", "gbla_reduce_C", "gbla_update_D", "gbla_echelon_D", "gbla_reduce",
            "gbla_get_dims", "gbla_get_maps", "gbla_get_D", "gbla_get_Cprime", "gbla_get_Bprime",
            "gbla_densify_quadrant", "gbla_get_rref", "gbla_copy_rref_to_host", "gbla_get_opcount",
            "gbla_get_phase_ms", "gbla_sync", "gbla_mat_free", "gbla_last_error", "gbla_version",
            "gbla_kernel_launches", "gbla_nccl_get_unique_id", "gbla_modgemm", "gbla_get_kernel_ms",
            "gbla_get_multilines", "gbla_get_kernel_work", "gbla_get_kernel_exec", "gbla_modgemm_bench", "gbla_rref_M", "gbla_get_rref_M",
            "gbla_file_info_parse", "gbla_file_decode", "gbla_get_multiline_runs", "gbla_reduce_wide",
            "gbla_get_wide"]


def _check(status: int):
    if status != 0:
        msg = _lib.gbla_last_error()
        raise GblaError(status, msg.decode() if msg else "")


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class _DevView:
    """__cuda_array_interface__ wrapper so torch can view library memory."""

    def __init__(self, ptr, shape, typestr, strides=None):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3,
                                         "strides": strides}


def _view(ptr, shape, dtype_str, ld=None, itemsize=None):
    import torch
    strides = None
    if ld is not None and len(shape) == 2:
        strides = (ld * itemsize, itemsize)
    if ptr is None or ptr == 0 or any(s == 0 for s in shape):
        tdt = {"<u2": torch.uint16, "<u4": torch.uint32, "<u8": torch.uint64}[dtype_str]
        return torch.zeros(shape, dtype=tdt, device="cuda")
    return torch.as_tensor(_DevView(ptr, shape, dtype_str, strides), device="cuda")


class Context:
    """A libgbla context on one CUDA device; device memory comes from torch."""

    def __init__(self, device: int = 0, torch_allocator: bool = True):
        import torch
        L = load_library()
        self._h = ctypes.c_void_p()
        _check(L.gbla_ctx_create(device, ctypes.byref(self._h)))
        self.device = device
        self._live = {}
        if torch_allocator:
            dev = torch.device("cuda", device)

            raw_alloc = torch.cuda.caching_allocator_alloc
            raw_free = torch.cuda.caching_allocator_delete

            def _alloc(nbytes, stream, user):
                # an exception must not cross the C boundary: out of memory -> NULL -> GBLA_E_NOMEM.
                # torch's caching allocator with the library's stream (a freed block is reused only in
                # that stream's order), not torch's current stream
                try:
                    ptr = int(raw_alloc(int(nbytes), device, int(stream or 0)))
                except Exception:
                    return None
                self._live[ptr] = True
                return ptr

            def _free(ptr, stream, user):
                if ptr and self._live.pop(int(ptr), None):
                    raw_free(int(ptr))

            self._alloc_cb = _ALLOC_FN(_alloc)
            self._free_cb = _FREE_FN(_free)
            _check(L.gbla_ctx_set_allocator(self._h, self._alloc_cb, self._free_cb, None))

            def _memq(user):
                # what torch can still hand out in one piece: its unused cached blocks go back to the
                # driver first (they may be fragmented), then the driver's free memory.  Called only
                # when the driver's free memory alone is short of a whole sparse phase's X tiles (c4),
                # never on a hot path: emptying the cache makes later allocations fresh cudaMallocs.
                try:
                    torch.cuda.empty_cache()
                    return int(torch.cuda.mem_get_info(dev)[0])
                except Exception:
                    return 0

            self._memq_cb = _MEMQ_FN(_memq)
            _check(L.gbla_ctx_set_mem_query(self._h, self._memq_cb, None))

    def set_comm(self, unique_id, rank: int, world: int):
        """gbla_ctx_set_comm; unique_id None detaches (world 1)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128) if unique_id is not None else None
        _check(_lib.gbla_ctx_set_comm(self._h, buf, rank, world))

    def close(self):
        if self._h:
            _lib.gbla_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(L.gbla_nccl_get_unique_id(buf))
    return buf.raw


class Mat:
    """A spliced matrix (gbla_mat) and its results."""

    def __init__(self, ctx: Context, handle, p: int, keep=()):
        self.ctx = ctx
        self._h = handle
        self.p = p
        self._keep = keep

    # ---- results
    def dims(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.gbla_get_dims(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def maps(self):
        """(sigma[n], pivot_row[npiv], nonpivot_row[mN]) as new torch tensors (int64)."""
        npiv, mN, nN = self.dims()
        s, pr, nr = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(_lib.gbla_get_maps(self._h, ctypes.byref(s), ctypes.byref(pr), ctypes.byref(nr)))
        return (_view(s.value, (npiv + nN,), "<u4").clone(), _view(pr.value, (npiv,), "<u4").clone(),
                _view(nr.value, (mN,), "<u4").clone())

    def D(self, clone: bool = True):
        """Current D (mN x nN).  clone=False returns a view of the library's
        buffer (valid until the next call on this handle changes it)."""
        npiv, mN, nN = self.dims()
        d, ld = ctypes.c_void_p(), ctypes.c_int64()
        _check(_lib.gbla_get_D(self._h, ctypes.byref(d), ctypes.byref(ld)))
        v = _view(d.value, (mN, nN), "<u2", ld.value, 2)
        return v.clone() if clone else v

    def cprime(self):
        npiv, mN, nN = self.dims()
        d, ld = ctypes.c_void_p(), ctypes.c_int64()
        _check(_lib.gbla_get_Cprime(self._h, ctypes.byref(d), ctypes.byref(ld)))
        return None if not d.value else _view(d.value, (mN, npiv), "<u2", ld.value, 2).clone()

    def bprime(self):
        npiv, mN, nN = self.dims()
        d, ld = ctypes.c_void_p(), ctypes.c_int64()
        _check(_lib.gbla_get_Bprime(self._h, ctypes.byref(d), ctypes.byref(ld)))
        return None if not d.value else _view(d.value, (npiv, nN), "<u2", ld.value, 2).clone()

    def quadrant(self, which: str, stream=None):
        import torch
        npiv, mN, nN = self.dims()
        shape = {"A": (npiv, npiv), "B": (npiv, nN), "C": (mN, npiv), "D": (mN, nN)}[which]
        ld = max(shape[1], 1)
        out = torch.zeros((max(shape[0], 1), ld), dtype=torch.uint16, device="cuda")
        _check(_lib.gbla_densify_quadrant(self._h, which.encode(), ctypes.c_void_p(out.data_ptr()), ld,
                                          _stream_ptr(stream)))
        torch.cuda.current_stream().synchronize()
        return out[:shape[0], :shape[1]]

    def multilines(self, stream=None):
        """Two-row multilines of A|B: (ptr[npairs+1], col[slots],
        val[slots]) as new torch tensors; val packs row 2k (low 16 bits) and
        row 2k+1 (high 16 bits)."""
        npr, ptr, col, val = ctypes.c_int64(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(_lib.gbla_get_multilines(self._h, _stream_ptr(stream), ctypes.byref(npr), ctypes.byref(ptr),
                                        ctypes.byref(col), ctypes.byref(val)))
        P = _view(ptr.value, (npr.value + 1,), "<u8").clone()
        ns = int(P[-1].item()) if npr.value >= 0 else 0
        return P, _view(col.value, (ns,), "<u4").clone(), _view(val.value, (ns,), "<u4").clone()

    def wide(self):
        """gbla_reduce_wide results: (rank, pivcol[rank], R[rank x nN], D_new[mN x nN]) as new torch
        tensors (uint32)."""
        npiv, mN, nN = self.dims()
        rk, pc, R, Dn, ld = (ctypes.c_int64(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(),
                             ctypes.c_int64())
        _check(_lib.gbla_get_wide(self._h, ctypes.byref(rk), ctypes.byref(pc), ctypes.byref(R), ctypes.byref(Dn),
                                  ctypes.byref(ld)))
        r = rk.value
        return (r, _view(pc.value, (r,), "<u4").clone(), _view(R.value, (r, nN), "<u4", ld.value, 4).clone(),
                _view(Dn.value, (mN, nN), "<u4", ld.value, 4).clone())

    def multiline_runs(self, stream=None):
        """Column runs of the multilines (gbla_get_multiline_runs): (run_ptr[npairs+1], run_col,
        run_len, run_slot) as new torch tensors."""
        nr, ptr, col, ln, sl = (ctypes.c_int64(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(),
                                ctypes.c_void_p())
        _check(_lib.gbla_get_multiline_runs(self._h, _stream_ptr(stream), ctypes.byref(nr), ctypes.byref(ptr),
                                            ctypes.byref(col), ctypes.byref(ln), ctypes.byref(sl)))
        npairs = (self.dims()[0] + 1) // 2
        n = nr.value
        return (_view(ptr.value, (npairs + 1,), "<u8").clone(), _view(col.value, (n,), "<u4").clone(),
                _view(ln.value, (n,), "<u4").clone(), _view(sl.value, (n,), "<u4").clone())

    def rank(self):
        """rank(D) (no copy of R)."""
        rk = ctypes.c_int64()
        _check(_lib.gbla_get_rref(self._h, ctypes.byref(rk), None, None, None))
        return rk.value

    def rref(self):
        """(rank, pivcol[rank], R[rank x nN]) as new torch tensors."""
        npiv, mN, nN = self.dims()
        rk, pc, R, ld = ctypes.c_int64(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
        _check(_lib.gbla_get_rref(self._h, ctypes.byref(rk), ctypes.byref(pc), ctypes.byref(R), ctypes.byref(ld)))
        r = rk.value
        return r, _view(pc.value, (r,), "<u4").clone(), _view(R.value, (r, nN), "<u2", ld.value, 2).clone()

    def rref_M(self, stream=None):
        """SURVEY 8(f) f2 (gbla_rref_M): RREF of the whole M in M's original column order, as
        (rank(M), row_ptr, col, val) new torch tensors (a CSR; rows sorted by pivot column)."""
        rk = ctypes.c_int64()
        _check(_lib.gbla_rref_M(self._h, _stream_ptr(stream), ctypes.byref(rk)))
        c = _CSR()
        _check(_lib.gbla_get_rref_M(self._h, ctypes.byref(c)))
        r, nnz = c.m, c.nnz
        return (r, _view(c.row_ptr, (r + 1,), "<u8").clone(), _view(c.col, (nnz,), "<u4").clone(),
                _view(c.val, (nnz,), "<u2").clone())

    def rref_to_host(self, stream=None, out=None):
        """(rank, pivcol, R) copied to host numpy arrays by the library.  `out` = (pivcol, R)
        host arrays to fill (e.g. views of pinned buffers), at least rank and rank x nN."""
        npiv, mN, nN = self.dims()
        rk = ctypes.c_int64()
        _check(_lib.gbla_get_rref(self._h, ctypes.byref(rk), None, None, None))
        r = rk.value
        if out is not None:
            pc, R = out
            if pc.size < r or R.shape[0] < r or R.shape[1] != max(nN, 1) or not R.flags.c_contiguous:
                raise ValueError("rref_to_host: output buffers too small or not contiguous rank x nN")
        else:
            pc = np.zeros(max(r, 1), np.uint32)
            R = np.zeros((max(r, 1), max(nN, 1)), np.uint16)
        _check(_lib.gbla_copy_rref_to_host(self._h, pc.ctypes.data_as(ctypes.c_void_p),
                                           R.ctypes.data_as(ctypes.c_void_p), _stream_ptr(stream)))
        return r, pc[:r], R[:r, :nN]

    def opcount(self):
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.gbla_get_opcount(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    KERNELS = ("sweep", "update", "panel", "trailing", "rnew", "backsub")

    def kernel_ms(self):
        """{family: (ms, launches)} from the library's CUDA-event timers
        (non-empty only if GBLA_KERNEL_TIMERS was set at handle creation)."""
        out = {}
        for i, name in enumerate(self.KERNELS):
            ms, n = ctypes.c_float(), ctypes.c_int64()
            _check(_lib.gbla_get_kernel_ms(self._h, i, ctypes.byref(ms), ctypes.byref(n)))
            out[name] = (ms.value, n.value)
        return out

    def kernel_work(self):
        """{family: algorithmic modMACs} (gbla_get_kernel_work)."""
        out = {}
        for i, name in enumerate(self.KERNELS):
            w = ctypes.c_uint64()
            _check(_lib.gbla_get_kernel_work(self._h, i, ctypes.byref(w)))
            out[name] = w.value
        w = ctypes.c_uint64()
        _check(_lib.gbla_get_kernel_work(self._h, len(self.KERNELS), ctypes.byref(w)))
        out["trailing_elems"] = w.value                 # D entries read + written by the trailing updates
        return out

    def kernel_exec(self):
        """{family: u8 MACs the tensor cores executed} (gbla_get_kernel_exec; 0 = not counted)."""
        out = {}
        for i, name in enumerate(self.KERNELS):
            w = ctypes.c_uint64()
            _check(_lib.gbla_get_kernel_exec(self._h, i, ctypes.byref(w)))
            out[name] = w.value
        return out

    def phase_ms(self):
        arr = (ctypes.c_float * 5)()
        _check(_lib.gbla_get_phase_ms(self._h, arr))
        return dict(zip(["splice", "reduce_C", "reduce_B", "update_D", "echelon"], list(arr)))

    def free(self):
        if self._h:
            _lib.gbla_mat_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _csr_struct(m, n, row_ptr, col, val):
    """Marshal a CSR given as torch CUDA tensors (device) or numpy arrays (host)."""
    host = isinstance(row_ptr, np.ndarray)
    if host:
        row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
        col = np.ascontiguousarray(col, np.uint32)
        val = np.ascontiguousarray(val, np.uint16)
        ptrs = [a.ctypes.data for a in (row_ptr, col, val)]
        nnz = int(row_ptr[-1]) if row_ptr.size else 0
        keep = (row_ptr, col, val)
    else:
        import torch
        for t, dt in ((row_ptr, torch.uint64), (col, torch.uint32), (val, torch.uint16)):
            if not t.is_cuda or t.dtype != dt or not t.is_contiguous():
                raise TypeError("device CSR must be contiguous CUDA tensors of dtypes uint64/uint32/uint16")
        ptrs = [t.data_ptr() for t in (row_ptr, col, val)]
        nnz = int(col.numel())
        keep = (row_ptr, col, val)
    return _CSR(m, n, nnz, ptrs[0], ptrs[1], ptrs[2]), host, keep


# ---- the six calls ------------------------------------------------------
def gbla_splice(ctx: Context, m, n, row_ptr, col, val, p, stream=None) -> Mat:
    """Step 1.  CSR arrays: torch CUDA tensors or numpy (host)."""
    csr, host, keep = _csr_struct(m, n, row_ptr, col, val)
    h = ctypes.c_void_p()
    _check(_lib.gbla_splice(ctx._h, ctypes.byref(csr), p, GBLA_HOST_INPUT if host else 0, _stream_ptr(stream),
                            ctypes.byref(h)))
    return Mat(ctx, h, p, keep)


def gbla_reduce_B(mat: Mat, stream=None):
    _check(_lib.gbla_reduce_B(mat._h, _stream_ptr(stream)))


def gbla_reduce_C(mat: Mat, fused: bool = True, keep_cprime: bool = False, int_pipe: bool = False, stream=None):
    """C <- C A^-1 (new order); fused: also D <- D - C A^-1 B.  int_pipe selects
    the per-target multiline AXPY kernel (GBLA_SPARSE_INT) instead of the
    tensor-core block path."""
    flags = (GBLA_FUSE_D if fused else 0) | (GBLA_KEEP_CPRIME if keep_cprime else 0)
    flags |= GBLA_SPARSE_INT if int_pipe else 0
    _check(_lib.gbla_reduce_C(mat._h, flags, _stream_ptr(stream)))


def gbla_update_D(mat: Mat, stream=None):
    _check(_lib.gbla_update_D(mat._h, _stream_ptr(stream)))


def gbla_echelon_D(mat: Mat, flags: int = 0, stream=None) -> int:
    r = ctypes.c_int64()
    _check(_lib.gbla_echelon_D(mat._h, flags, _stream_ptr(stream), ctypes.byref(r)))
    return r.value


def gbla_reduce(ctx: Context, m, n, row_ptr, col, val, p, flags: int = 0, stream=None) -> Mat:
    """Whole pipeline (new order by default).  Host numpy input => the library
    copies it to the device (GBLA_HOST_INPUT)."""
    csr, host, keep = _csr_struct(m, n, row_ptr, col, val)
    h = ctypes.c_void_p()
    _check(_lib.gbla_reduce(ctx._h, ctypes.byref(csr), p, flags | (GBLA_HOST_INPUT if host else 0),
                            _stream_ptr(stream), ctypes.byref(h)))
    return Mat(ctx, h, p, keep)


def gbla_modgemm(ctx: Context, p: int, A, B, C, rowidx=None, engine: int = 0, stream=None):
    """K11: C[rowidx[i]] -= A[i] @ B  (mod p), in place.  A: rows x K, B: K x cols,
    C: torch uint16 CUDA tensors (2-D, unit column stride); K <= 512."""
    rows, K = A.shape
    K2, cols = B.shape
    assert K == K2 and C.shape[1] >= cols
    ri = ctypes.c_void_p(rowidx.data_ptr()) if rowidx is not None else None
    _check(_lib.gbla_modgemm(ctx._h, p, rows, cols, K, ctypes.c_void_p(A.data_ptr()), A.stride(0),
                             ctypes.c_void_p(B.data_ptr()), B.stride(0), ri, ctypes.c_void_p(C.data_ptr()),
                             C.stride(0), engine, _stream_ptr(stream)))


def gbla_reduce_wide(ctx: Context, m, n, row_ptr, col, val, p, stream=None) -> Mat:
    """the reduction over GF(p) for a prime 2 < p < 2^31 (gbla_reduce_wide).  CSR
    arrays: numpy (host: row_ptr u64, col u32, val u32) or torch CUDA tensors (uint64/uint32/uint32).
    Results: Mat.wide() -> (rank, pivcol, R, D_new); dims / maps / opcount as for gbla_reduce."""
    host = isinstance(row_ptr, np.ndarray)
    if host:
        row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
        col = np.ascontiguousarray(col, np.uint32)
        val = np.ascontiguousarray(val, np.uint32)
        ptrs = [a.ctypes.data for a in (row_ptr, col, val)]
        nnz = int(row_ptr[-1]) if row_ptr.size else 0
    else:
        ptrs = [t.data_ptr() for t in (row_ptr, col, val)]
        nnz = int(col.numel())
    keep = (row_ptr, col, val)
    csr = _CSR(m, n, nnz, ptrs[0], ptrs[1], ptrs[2])       # same layout as gbla_csr32 (val: u32 pointer)
    h = ctypes.c_void_p()
    _check(_lib.gbla_reduce_wide(ctx._h, ctypes.byref(csr), p, GBLA_HOST_INPUT if host else 0,
                                 _stream_ptr(stream), ctypes.byref(h)))
    return Mat(ctx, h, p, keep)


def modgemm_bench(ctx: Context, p: int, rows: int, cols: int, K: int, reps: int = 10, stream=None) -> float:
    """K11 microbenchmark (gbla_modgemm_bench): mean device ms per launch of
    C -= A B mod p on device-generated operands (rows x cols, K <= 512)."""
    ms = ctypes.c_float()
    _check(_lib.gbla_modgemm_bench(ctx._h, p, rows, cols, K, reps, _stream_ptr(stream), ctypes.byref(ms)))
    return ms.value


def file_info(data: bytes, fmt: int) -> dict:
    """gbla_file_info_parse: the header of a Format 1 / Format 2 file image."""
    fi = _FileInfo()
    buf = ctypes.create_string_buffer(bytes(data), len(data))
    _check(load_library().gbla_file_info_parse(buf, len(data), fmt, ctypes.byref(fi)))
    return {k: getattr(fi, k) for k, _ in _FileInfo._fields_}


def file_decode(ctx: Context, data: bytes, fmt: int, stream=None):
    """gbla_file_decode: decode a file image on the device.  Returns (m, n, p, row_ptr, col, val)
    with new torch CUDA tensors (uint64 / uint32 / uint16), ready for gbla_splice / gbla_reduce."""
    import torch
    info = file_info(data, fmt)
    m, nnz = info["m"], info["nnz"]
    rp = torch.empty(m + 1, dtype=torch.uint64, device="cuda")
    col = torch.empty(max(nnz, 1), dtype=torch.uint32, device="cuda")
    val = torch.empty(max(nnz, 1), dtype=torch.uint16, device="cuda")
    buf = ctypes.create_string_buffer(bytes(data), len(data))
    _check(_lib.gbla_file_decode(ctx._h, buf, len(data), fmt, ctypes.c_void_p(rp.data_ptr()),
                                 ctypes.c_void_p(col.data_ptr()), ctypes.c_void_p(val.data_ptr()),
                                 _stream_ptr(stream)))
    return m, info["n"], info["p"], rp, col[:nnz], val[:nnz]


def tile_shard(ntiles: int, rank: int, world: int):
    """Target tiles owned by `rank` in the multi-GPU sparse phase (dist.cu):
    tiles are dealt cyclically, T = rank, rank + world, ...  (pure mirror of
    the library's partition, for tests and reporting)."""
    return list(range(rank, ntiles, world))


def kernel_launches() -> int:
    return int(load_library().gbla_kernel_launches())


def version() -> str:
    return load_library().gbla_version().decode()

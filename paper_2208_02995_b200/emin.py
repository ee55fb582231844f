"""Thin ctypes binding of libemin.so (the C ABI in include/emin.h).

Argument marshalling only: every step of the method runs in the CUDA kernels
behind the ABI.  There is no fallback: if libemin.so is missing or no CUDA
device is present, the calls raise.

Arrays are numpy (host) or torch tensors.  If the A/P/B arrays are CUDA
tensors the library reads them in place (``inputs_on_device = 1``); host
arrays are copied by ``emin_setup`` itself (that copy is part of the C call).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libemin.so")
_lib = None

STATUS = ["EMIN_OK", "EMIN_ERR_ARG", "EMIN_ERR_CSR", "EMIN_ERR_PATTERN", "EMIN_ERR_BC",
          "EMIN_ERR_DIAG", "EMIN_ERR_NONFINITE", "EMIN_ERR_BREAKDOWN", "EMIN_ERR_CUDA",
          "EMIN_ERR_NCCL", "EMIN_ERR_OOM", "EMIN_ERR_STATE"]
STOP_REASONS = {0: "running", 1: "gamma<=0", 2: "y'Ky==0", 3: "tau", 4: "stagnation",
                5: "breakdown"}
KERNEL_PATHS = {0: "generic", 1: "scalar", 2: "nodal3"}


class EminError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS[code] if 0 <= code < len(STATUS) else code}: {msg}")
        self.code = code


class emin_opts(C.Structure):
    _fields_ = [("block_size", C.c_int32), ("rank_tol", C.c_double), ("tau", C.c_double),
                ("project_after_jacobi", C.c_int32), ("stagnation_rel", C.c_double),
                ("stream", C.c_void_p), ("nccl_comm", C.c_void_p),
                ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("inputs_on_device", C.c_int32), ("precond", C.c_int32), ("sgs_key", C.c_void_p),
                ("start", C.c_int32), ("loopback", C.c_void_p), ("loopback_rank", C.c_int32),
                ("debug_flags", C.c_int32)]


# emin_opts.debug_flags bits (include/emin.h): alternative kernel paths for tests / A/B
DBG_FORCE_GENERIC, DBG_NO_R0E, DBG_SGS_GENERIC, DBG_TRACE, DBG_FUSE_SCALARS, DBG_ALG2_ROWS = 1, 2, 4, 8, 16, 32
DBG_AB1 = 64
DBG_AB2 = 128
DBG_UNSCALED = 512
GALERKIN_DEVICE, GALERKIN_POINT = 1, 2


EMIN_PREC_JACOBI, EMIN_PREC_SGS = 0, 1
PRECONDS = {"jacobi": EMIN_PREC_JACOBI, "sgs": EMIN_PREC_SGS}
EMIN_START_GIVEN, EMIN_START_MAXVOL = 0, 1
STARTS = {"given": EMIN_START_GIVEN, "maxvol": EMIN_START_MAXVOL}


class emin_report_t(C.Structure):
    _fields_ = [("E0", C.c_double), ("dE1", C.c_double), ("k_total", C.c_int64),
                ("stop_reason", C.c_int32), ("n_svd_rows", C.c_int64),
                ("n_frozen_rows", C.c_int64), ("n_fine", C.c_int64), ("nnz_W", C.c_int64),
                ("nnz_AFF", C.c_int64), ("kernel_path", C.c_int32), ("nranks", C.c_int32),
                ("launches", C.c_int64), ("precond", C.c_int32), ("sgs_levels", C.c_int64),
                ("n_maxvol_fail", C.c_int64), ("rank", C.c_int32), ("n_halo_rows", C.c_int64),
                ("n_halo_entries", C.c_int64), ("n_send_entries", C.c_int64),
                ("n_interior_units", C.c_int64)]


EXPORTED = ["emin_default_opts", "emin_setup", "emin_iterate", "emin_energy", "emin_get_P",
            "emin_reset", "emin_report", "emin_destroy", "emin_status_str", "emin_last_error",
            "emin_set_profiling", "emin_kernel_times", "emin_get_layout", "emin_nccl_unique_id",
            "emin_nccl_comm_init", "emin_nccl_comm_destroy", "emin_pattern", "emin_pattern_error",
            "emin_galerkin", "emin_galerkin_error", "emin_galerkin_path", "emin_loopback_create",
            "emin_loopback_destroy", "emin_release_memory"]


def load_library():
    """Load libemin.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not found: run __graft_entry__.build() "
                           "(the CUDA path has no fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
    lib.emin_default_opts.argtypes = [C.POINTER(emin_opts), i64]
    lib.emin_default_opts.restype = None
    lib.emin_setup.argtypes = [C.POINTER(P), i64, i64, P, P, P, P, P, P, P, i32, P, P,
                               C.POINTER(emin_opts)]
    lib.emin_setup.restype = i32
    lib.emin_iterate.argtypes = [P, i32, C.POINTER(i32), P]
    lib.emin_iterate.restype = i32
    lib.emin_energy.argtypes = [P, C.POINTER(dbl)]
    lib.emin_energy.restype = i32
    lib.emin_get_P.argtypes = [P, P]
    lib.emin_get_P.restype = i32
    lib.emin_reset.argtypes = [P]
    lib.emin_reset.restype = i32
    lib.emin_report.argtypes = [P, C.POINTER(emin_report_t)]
    lib.emin_report.restype = i32
    lib.emin_destroy.argtypes = [P]
    lib.emin_destroy.restype = None
    lib.emin_status_str.argtypes = [i32]
    lib.emin_status_str.restype = C.c_char_p
    lib.emin_last_error.argtypes = [P]
    lib.emin_last_error.restype = C.c_char_p
    lib.emin_set_profiling.argtypes = [P, i32]
    lib.emin_set_profiling.restype = i32
    lib.emin_kernel_times.argtypes = [P, P, P]
    lib.emin_kernel_times.restype = i32
    lib.emin_get_layout.argtypes = [P, P, P, P]
    lib.emin_get_layout.restype = i32
    lib.emin_nccl_unique_id.argtypes = [P]
    lib.emin_nccl_unique_id.restype = i32
    lib.emin_nccl_comm_init.argtypes = [C.POINTER(P), i32, P, i32]
    lib.emin_nccl_comm_init.restype = i32
    lib.emin_nccl_comm_destroy.argtypes = [P]
    lib.emin_nccl_comm_destroy.restype = i32
    lib.emin_pattern.argtypes = [i64, P, P, P, i32, i32, P, i64, i32, i32, P, P, i64, C.POINTER(i64), i32, P]
    lib.emin_pattern.restype = i32
    lib.emin_pattern_error.argtypes = []
    lib.emin_pattern_error.restype = C.c_char_p
    lib.emin_galerkin.argtypes = [i64, i64, P, P, P, P, P, P, P, P, P, i64, C.POINTER(i64), i32, P]
    lib.emin_galerkin.restype = i32
    lib.emin_galerkin_error.argtypes = []
    lib.emin_galerkin_error.restype = C.c_char_p
    lib.emin_galerkin_path.argtypes = []
    lib.emin_galerkin_path.restype = i32
    lib.emin_loopback_create.argtypes = [C.POINTER(P), i32]
    lib.emin_loopback_create.restype = i32
    lib.emin_loopback_destroy.argtypes = [P]
    lib.emin_loopback_destroy.restype = None
    lib.emin_release_memory.argtypes = []
    lib.emin_release_memory.restype = None
    _lib = lib
    return lib


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _check(st, ctx_handle=None):
    if st != 0:
        lib = load_library()
        msg = lib.emin_last_error(ctx_handle).decode()
        raise EminError(st, msg)


def _prep(a, np_dtype, torch_dtype=None):
    if a is None:
        return None
    if _is_torch(a):
        import torch
        t = a.contiguous()
        if torch_dtype is not None and t.dtype != torch_dtype:
            raise TypeError(f"expected {torch_dtype}, got {t.dtype}")
        return t
    return np.ascontiguousarray(a, dtype=np_dtype)


# ---------------------------------------------------------------------------
# the ABI calls, same names
# ---------------------------------------------------------------------------

def emin_setup(n_global, nc_global, A_rowptr, A_col, A_val, is_coarse, P_rowptr, P_col, P_val,
               nv, B, Bc, *, block_size=1, rank_tol=1e-10, tau=0.0, project_after_jacobi=0,
               stagnation_rel=1e-30, stream=None, nccl_comm=None, row_begin=0, row_end=None,
               precond="jacobi", sgs_key=None, start="given", loopback=None, loopback_rank=0,
               debug_flags=0):
    """emin_setup (include/emin.h).  Returns the opaque context handle.
    precond: "jacobi" | "sgs" (or EMIN_PREC_*); sgs_key: per owned row,
    same side (host / cuda) as the other arrays, or None.  start: "given"
    (P_val / least-norm) or "maxvol" (Alg. 1's tentative start).
    loopback / loopback_rank: an emin_loopback_create handle and this
    context's rank in it (R contexts on one device, one thread each).
    debug_flags: EMIN_DBG_* bits (alternative kernel paths for tests)."""
    lib = load_library()
    import torch
    arrs = [A_rowptr, A_col, A_val, is_coarse, P_rowptr, P_col, P_val, B, Bc]
    on_dev = [_is_torch(a) and a.is_cuda for a in arrs if a is not None]
    if any(on_dev) and not all(on_dev):
        raise ValueError("all arrays must be on the same side (host or cuda)")
    dev = bool(on_dev and all(on_dev))
    tdt = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64,
           np.uint8: torch.uint8}
    keep = [_prep(a, dt, tdt[dt] if dev else None) for a, dt in
            zip(arrs, [np.int64, np.int32, np.float64, np.uint8, np.int64, np.int32, np.float64,
                       np.float64, np.float64])]
    key = None
    if sgs_key is not None:
        if dev and not (_is_torch(sgs_key) and sgs_key.is_cuda):
            sgs_key = torch.from_numpy(np.ascontiguousarray(sgs_key, dtype=np.int64)).cuda()
        key = _prep(sgs_key, np.int64, torch.int64 if dev else None)
    o = emin_opts()
    lib.emin_default_opts(C.byref(o), int(n_global))
    o.block_size = block_size
    o.rank_tol = rank_tol
    o.tau = tau
    o.project_after_jacobi = project_after_jacobi
    o.stagnation_rel = stagnation_rel
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    o.stream = C.c_void_p(int(stream))
    o.nccl_comm = nccl_comm
    o.row_begin = row_begin
    o.row_end = n_global if row_end is None else row_end
    o.inputs_on_device = 1 if dev else 0
    o.precond = PRECONDS[precond] if isinstance(precond, str) else int(precond)
    o.sgs_key = _ptr(key)
    o.start = STARTS[start] if isinstance(start, str) else int(start)
    o.loopback = loopback
    o.loopback_rank = int(loopback_rank)
    o.debug_flags = int(debug_flags)
    h = C.c_void_p()
    st = lib.emin_setup(C.byref(h), int(n_global), int(nc_global), *[_ptr(a) for a in keep[:7]],
                        int(nv), _ptr(keep[7]), _ptr(keep[8]), C.byref(o))
    if st != 0:
        raise EminError(st, lib.emin_last_error(None).decode())
    return h


def emin_iterate(ctx, k, want=False):
    """Run up to k steps.  want=True returns (k_done, dE ndarray) and syncs."""
    lib = load_library()
    if want:
        kd = C.c_int32(0)
        dE = np.zeros(max(int(k), 1))
        _check(lib.emin_iterate(ctx, int(k), C.byref(kd), dE.ctypes.data_as(C.c_void_p)), ctx)
        return kd.value, dE[:kd.value].copy()
    _check(lib.emin_iterate(ctx, int(k), None, None), ctx)
    return None


def emin_energy(ctx):
    lib = load_library()
    E = C.c_double(0.0)
    _check(lib.emin_energy(ctx, C.byref(E)), ctx)
    return E.value


def emin_get_P(ctx, out):
    """Write the owned P values into ``out`` (numpy array or cuda tensor,
    float64, input CSR order; device only if the context was set up from
    device arrays)."""
    lib = load_library()
    _check(lib.emin_get_P(ctx, _ptr(out)), ctx)
    return out


def emin_reset(ctx):
    _check(load_library().emin_reset(ctx), ctx)


def emin_report(ctx):
    rep = emin_report_t()
    _check(load_library().emin_report(ctx, C.byref(rep)), ctx)
    return {f: getattr(rep, f) for f, _ in rep._fields_}


def emin_destroy(ctx):
    if ctx is not None:
        load_library().emin_destroy(ctx)


def emin_get_layout(ctx):
    rep = emin_report(ctx)
    nF, W = rep["n_fine"], rep["nnz_W"]
    wptr = np.empty(nF + 1, np.int64)
    wcol = np.empty(max(W, 1), np.int32)
    pofs = np.empty(max(nF, 1), np.int64)
    _check(load_library().emin_get_layout(ctx, _ptr(wptr), _ptr(wcol), _ptr(pofs)), ctx)
    return wptr, wcol[:W], pofs[:nF]


def emin_pattern(n, A_rowptr, A_col, is_coarse, block_size, nv, Bc, nc, l0=2, lmax=4, stream=None):
    """emin_pattern (include/emin.h): Alg. 1's pattern growth from the graph
    of A on the GPU.  Inputs all host numpy arrays (returns numpy) or all
    CUDA tensors (returns CUDA tensors); returns (P_rowptr, P_col)."""
    lib = load_library()
    import torch
    dev = _is_torch(A_rowptr)
    if dev:
        arrs = [A_rowptr.to(torch.int64).contiguous(), A_col.to(torch.int32).contiguous(),
                is_coarse.to(torch.uint8).contiguous(), Bc.to(torch.float64).contiguous()]
        rp = torch.zeros(int(n) + 1, dtype=torch.int64, device=A_rowptr.device)
    else:
        arrs = [np.ascontiguousarray(A_rowptr, np.int64), np.ascontiguousarray(A_col, np.int32),
                np.ascontiguousarray(is_coarse, np.uint8), np.ascontiguousarray(Bc, np.float64)]
        rp = np.zeros(int(n) + 1, np.int64)
    nnz = C.c_int64(0)
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    st = lib.emin_pattern(int(n), _ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), int(block_size), int(nv),
                          _ptr(arrs[3]), int(nc), int(l0), int(lmax), _ptr(rp), None, 0, C.byref(nnz),
                          int(dev), C.c_void_p(int(stream)))
    if st != 0:
        raise EminError(st, lib.emin_pattern_error().decode())
    m = max(nnz.value, 1)
    col = torch.zeros(m, dtype=torch.int32, device=A_rowptr.device) if dev else np.zeros(m, np.int32)
    st = lib.emin_pattern(int(n), _ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), int(block_size), int(nv),
                          _ptr(arrs[3]), int(nc), int(l0), int(lmax), _ptr(rp), _ptr(col), nnz.value,
                          C.byref(nnz), int(dev), C.c_void_p(int(stream)))
    if st != 0:
        raise EminError(st, lib.emin_pattern_error().decode())
    return rp, col[:nnz.value]


def emin_galerkin(n, nc, A_rowptr, A_col, A_val, P_rowptr, P_col, P_val, stream=None, point=False):
    """emin_galerkin (include/emin.h): A_c = P^T A P on the GPU.  Inputs all
    host numpy arrays (returns numpy) or all CUDA tensors (returns CUDA
    tensors, nothing leaves the device but the nnz count).  point=True forces
    the point product (EMIN_GALERKIN_POINT)."""
    lib = load_library()
    import torch
    dev = _is_torch(A_rowptr)
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    if dev:
        arrs = [A_rowptr.to(torch.int64).contiguous(), A_col.to(torch.int32).contiguous(),
                A_val.to(torch.float64).contiguous(), P_rowptr.to(torch.int64).contiguous(),
                P_col.to(torch.int32).contiguous(), P_val.to(torch.float64).contiguous()]
        rp = torch.zeros(int(nc) + 1, dtype=torch.int64, device=A_rowptr.device)
    else:
        arrs = [np.ascontiguousarray(A_rowptr, np.int64), np.ascontiguousarray(A_col, np.int32),
                np.ascontiguousarray(A_val, np.float64), np.ascontiguousarray(P_rowptr, np.int64),
                np.ascontiguousarray(P_col, np.int32), np.ascontiguousarray(P_val, np.float64)]
        rp = np.zeros(int(nc) + 1, np.int64)
    nnz = C.c_int64(0)
    sp = C.c_void_p(int(stream))
    flags = (GALERKIN_DEVICE if dev else 0) | (GALERKIN_POINT if point else 0)
    st = lib.emin_galerkin(int(n), int(nc), *[_ptr(a) for a in arrs], _ptr(rp), None, None, 0, C.byref(nnz),
                           flags, sp)
    if st != 0:
        raise EminError(st, lib.emin_galerkin_error().decode())
    m = max(nnz.value, 1)
    if dev:
        col = torch.empty(m, dtype=torch.int32, device=A_rowptr.device)
        val = torch.empty(m, dtype=torch.float64, device=A_rowptr.device)
    else:
        col, val = np.zeros(m, np.int32), np.zeros(m, np.float64)
    st = lib.emin_galerkin(int(n), int(nc), *[_ptr(a) for a in arrs], _ptr(rp), _ptr(col), _ptr(val), m,
                           C.byref(nnz), flags, sp)
    if st != 0:
        raise EminError(st, lib.emin_galerkin_error().decode())
    return rp, col[:nnz.value], val[:nnz.value]


def emin_nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    _check(load_library().emin_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def emin_nccl_comm_init(nranks, uid, rank):
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    comm = C.c_void_p()
    _check(load_library().emin_nccl_comm_init(C.byref(comm), int(nranks), C.cast(buf, C.c_void_p), int(rank)))
    return comm


def emin_nccl_comm_destroy(comm):
    _check(load_library().emin_nccl_comm_destroy(comm))


def nccl_comm_from_torch(group=None):
    """Create an NCCL communicator for libemin over the ranks of a
    torch.distributed group (the unique id travels through torch)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [emin_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return emin_nccl_comm_init(world, obj[0], rank)


def emin_loopback_create(nranks):
    """In-process loopback group of ``nranks`` contexts (include/emin.h)."""
    h = C.c_void_p()
    _check(load_library().emin_loopback_create(C.byref(h), int(nranks)))
    return h


def emin_loopback_destroy(h):
    load_library().emin_loopback_destroy(h)


def emin_release_memory():
    load_library().emin_release_memory()


def emin_set_profiling(ctx, on):
    _check(load_library().emin_set_profiling(ctx, 1 if on else 0), ctx)


def emin_kernel_times(ctx):
    ms = np.zeros(4)
    n = np.zeros(4, np.int64)
    _check(load_library().emin_kernel_times(ctx, ms.ctypes.data_as(C.c_void_p),
                                            n.ctypes.data_as(C.c_void_p)), ctx)
    return {"stage1": (ms[0], int(n[0])), "stage2": (ms[1], int(n[1])),
            "spgemm": (ms[2], int(n[2])), "scalar": (ms[3], int(n[3]))}


# ---------------------------------------------------------------------------
# convenience wrapper
# ---------------------------------------------------------------------------

class Emin:
    """RAII-style wrapper around one context.

    ``Emin.from_problem(prob, device='cuda')`` stages a workloads.Problem
    (device='cuda': copied to the GPU by torch first, so emin_setup reads
    device memory; device='host': emin_setup copies from host memory)."""

    def __init__(self, handle, nnzP):
        self.h = handle
        self.nnzP = nnzP

    @classmethod
    def from_problem(cls, prob, device="cuda", **opts):
        import torch
        arrs = dict(A_rowptr=prob.A_rowptr, A_col=prob.A_col, A_val=prob.A_val,
                    is_coarse=prob.is_coarse, P_rowptr=prob.P_rowptr, P_col=prob.P_col,
                    P_val=prob.P_val, B=prob.B, Bc=prob.Bc)
        if device == "cuda":
            arrs = {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v)).cuda())
                    for k, v in arrs.items()}
        opts.setdefault("block_size", prob.block_size)
        h = emin_setup(prob.n, prob.nc, arrs["A_rowptr"], arrs["A_col"], arrs["A_val"],
                       arrs["is_coarse"], arrs["P_rowptr"], arrs["P_col"], arrs["P_val"],
                       prob.nv, arrs["B"], arrs["Bc"], **opts)
        obj = cls(h, int(prob.P_rowptr[-1]))
        obj._dev_inputs = device == "cuda"
        return obj

    def iterate(self, k, want=True):
        return emin_iterate(self.h, k, want)

    def energy(self):
        return emin_energy(self.h)

    def get_P(self):
        if getattr(self, "_dev_inputs", False):
            import torch
            out = torch.empty(self.nnzP, dtype=torch.float64, device="cuda")
            emin_get_P(self.h, out)
            return out.cpu().numpy()
        out = np.empty(self.nnzP)
        return emin_get_P(self.h, out)

    def reset(self):
        emin_reset(self.h)

    def layout(self):
        return emin_get_layout(self.h)

    def report(self):
        return emin_report(self.h)

    def close(self):
        if self.h is not None:
            emin_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

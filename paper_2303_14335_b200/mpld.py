"""Thin ctypes binding of the C ABI in include/mpld.h (argument marshalling only).

Every step of the decomposition runs in the CUDA kernels of lib/libmpld.so; this
module never computes any part of the result.  There is no CPU fallback: if the
library is missing or no CUDA device is present the calls raise.

Array arguments may be numpy arrays / torch CPU tensors (host entry points) or
torch CUDA tensors (device entry points).  Graph arrays and colours are int32,
counts and stats int64, costs float64 (include/mpld.h); torch tensors and
output buffers of another element type or not contiguous are rejected
(TypeError / ValueError), numpy inputs are converted.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPLD_LIB") or os.path.join(HERE, "lib", "libmpld.so")  # MPLD_LIB: tuning builds

MPLD_OK = 0
MPLD_ERR_ARG, MPLD_ERR_GRAPH, MPLD_ERR_COMPONENT, MPLD_ERR_CUDA, MPLD_ERR_NOMEM = 1, 2, 3, 4, 5
MPLD_FLAG_VALIDATE = 1
MPLD_FLAG_TILES = 2  # the tile pipeline (whole-graph pipeline gated behind it); identical results
MPLD_MAX_K = 4
MPLD_MAX_COMPONENT = 64
MPLD_COST_UNITS = 1000
STAT_NAMES = ["components", "hidden", "rounds", "max_component", "steps", "truncated", "error", "launches",
              "max_steps", "spill_refused"]
MPLD_STAT_LEN = len(STAT_NAMES)

# every symbol include/mpld.h declares
EXPORTS = ["mpld_last_error", "mpld_version", "mpld_decompose", "mpld_decompose_batch", "mpld_context_create",
           "mpld_context_destroy", "mpld_decompose_device", "mpld_context_set_timing",
           "mpld_context_reset_timing", "mpld_kernel_count", "mpld_kernel_name", "mpld_context_kernel_time",
           "mpld_context_debug", "mpld_prepare_device", "mpld_search_device", "mpld_finish_device",
           "mpld_decompose_batch_async", "mpld_decompose_batch_pairs_async", "mpld_wait",
           "mpld_shard_export", "mpld_shard_import", "mpld_decompose_batch_upper_async"]


class MPLDError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"mpld error {code}: {msg}")
        self.code = code


_lib = None
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


def lib():
    """Load lib/libmpld.so (raises OSError loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    L.mpld_last_error.restype = ctypes.c_char_p
    L.mpld_version.restype = ctypes.c_char_p
    L.mpld_kernel_name.restype = ctypes.c_char_p
    L.mpld_kernel_name.argtypes = [ctypes.c_int]
    L.mpld_kernel_count.restype = ctypes.c_int
    L.mpld_decompose.argtypes = [ctypes.c_int32, _vp, _vp, _vp, _vp, ctypes.c_int32, ctypes.c_double,
                                 ctypes.c_int64, _vp, _i64p, _i64p, _f64p]
    L.mpld_decompose_batch.argtypes = [ctypes.c_int32, _vp, ctypes.c_int32, _vp, _vp, _vp, _vp, ctypes.c_int32,
                                       ctypes.c_double, ctypes.c_int64, ctypes.c_uint32, _vp, _vp, _vp, _vp, _vp]
    L.mpld_context_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(_vp)]
    L.mpld_context_destroy.argtypes = [_vp]
    L.mpld_context_destroy.restype = None
    L.mpld_decompose_device.argtypes = [_vp, _vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp, _vp, _vp, _vp,
                                        ctypes.c_int32, ctypes.c_double, ctypes.c_int64, ctypes.c_uint32, _vp, _vp,
                                        _vp, _vp]
    L.mpld_context_set_timing.argtypes = [_vp, ctypes.c_int]
    L.mpld_context_reset_timing.argtypes = [_vp]
    L.mpld_context_kernel_time.argtypes = [_vp, ctypes.c_int, _f64p, _i64p]
    L.mpld_context_debug.argtypes = [_vp, _vp, ctypes.c_int]
    L.mpld_prepare_device.argtypes = [_vp, _vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp, _vp, _vp, _vp,
                                      ctypes.c_int32, ctypes.c_uint32, _vp, _vp]
    L.mpld_search_device.argtypes = [_vp, _vp, ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _vp]
    L.mpld_finish_device.argtypes = [_vp, _vp, ctypes.c_double, _vp, _vp, _vp, _vp]
    L.mpld_decompose_batch_async.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp, _vp, _vp, _vp,
                                             ctypes.c_int32, ctypes.c_double, ctypes.c_int64, ctypes.c_uint32, _vp,
                                             _vp, _vp, _vp, _vp, _i64p]
    L.mpld_decompose_batch_pairs_async.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp, _vp, ctypes.c_int64,
                                                   _vp, ctypes.c_int32, ctypes.c_double, ctypes.c_int64,
                                                   ctypes.c_uint32, _vp, _vp, _vp, _vp, _vp, _i64p]
    L.mpld_wait.argtypes = [_vp, ctypes.c_int64]
    L.mpld_shard_export.argtypes = [_vp, _vp, _vp, _vp, _vp]
    L.mpld_decompose_batch_upper_async.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp, ctypes.c_int64,
                                                   _vp, ctypes.c_int64, _vp, ctypes.c_int32, ctypes.c_double,
                                                   ctypes.c_int64, ctypes.c_uint32, _vp, _vp, _vp, _vp, _vp, _i64p]
    L.mpld_shard_import.argtypes = [_vp, _vp, _vp, ctypes.c_int64, _vp]
    _lib = L
    return L


def _check(rc: int):
    if rc != MPLD_OK:
        raise MPLDError(rc, lib().mpld_last_error().decode())


_TORCH_DTYPE = {np.dtype(np.int32): "torch.int32", np.dtype(np.int64): "torch.int64",
                np.dtype(np.float64): "torch.float64", np.dtype(np.uint8): "torch.uint8"}


def _check_tensor(t, dtype, what):
    """A torch tensor argument must have the element type the C ABI reads and be contiguous."""
    want = _TORCH_DTYPE[np.dtype(dtype)]
    if str(t.dtype) != want:
        raise TypeError(f"{what}: expected {want}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")


def _host_ptr(x, dtype=np.int32, what="host array"):
    """Address of a host input buffer (numpy array or torch CPU tensor) plus a
    keep-alive.  numpy inputs are converted to `dtype`; torch tensors must
    already have it (no silent reinterpretation of e.g. int64 indices)."""
    if hasattr(x, "data_ptr"):
        if x.is_cuda:
            raise ValueError(f"{what}: host entry point given a CUDA tensor")
        _check_tensor(x, dtype, what)
        return x.data_ptr(), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, a


def _out_ptr(x, dtype, what="host output"):
    """Address of a host output buffer (written in place: must be contiguous and
    of exactly the element type the C ABI writes)."""
    if hasattr(x, "data_ptr"):
        if x.is_cuda:
            raise ValueError(f"{what}: host outputs must be CPU tensors / arrays")
        _check_tensor(x, dtype, what)
        return x.data_ptr()
    if not isinstance(x, np.ndarray) or x.dtype != np.dtype(dtype) or not x.flags["C_CONTIGUOUS"]:
        raise TypeError(f"{what}: host outputs must be contiguous {np.dtype(dtype)} arrays")
    return x.ctypes.data


def _dev_ptr(t, dtype=np.int32, what="device tensor"):
    if t is None:
        return None
    if not (hasattr(t, "is_cuda") and t.is_cuda):
        raise ValueError(f"{what}: device entry point needs CUDA tensors")
    _check_tensor(t, dtype, what)
    return t.data_ptr()


# element types of the result buffers (include/mpld.h)
_OUT_DTYPES = {"colors": np.int32, "n_conflicts": np.int64, "n_stitches": np.int64, "cost": np.float64,
               "stats": np.int64}


def version() -> str:
    return lib().mpld_version().decode()


def mpld_decompose(n, ce_rowptr, ce_col, se_rowptr, se_col, k: int, alpha: float, max_steps: int = 0):
    """C ABI `mpld_decompose` on host buffers -> (colors, n_conflicts, n_stitches, cost)."""
    L = lib()
    colors = np.empty(max(int(n), 0), dtype=np.int32)
    nc, ns, cost = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    keep = [_host_ptr(a) for a in (ce_rowptr, ce_col, se_rowptr, se_col)]
    _check(L.mpld_decompose(int(n), *[p for p, _ in keep], int(k), float(alpha), int(max_steps),
                            colors.ctypes.data, ctypes.byref(nc), ctypes.byref(ns), ctypes.byref(cost)))
    return colors, nc.value, ns.value, cost.value


def mpld_decompose_batch(layout_offsets, n, ce_rowptr, ce_col, se_rowptr, se_col, k: int, alpha: float,
                         max_steps: int = 0, flags: int = 0, out_colors=None):
    """C ABI `mpld_decompose_batch` on host buffers -> dict with colors,
    per-layout n_conflicts / n_stitches / cost and stats."""
    L = lib()
    lo_p, lo = _host_ptr(layout_offsets)
    n_layouts = int(len(lo) - 1) if not hasattr(lo, "numel") else int(lo.numel() - 1)
    colors = out_colors if out_colors is not None else np.empty(max(int(n), 0), dtype=np.int32)
    col_p = _out_ptr(colors, np.int32, "out_colors")
    nc = np.zeros(n_layouts, dtype=np.int64)
    ns = np.zeros(n_layouts, dtype=np.int64)
    cost = np.zeros(n_layouts, dtype=np.float64)
    stats = np.zeros(MPLD_STAT_LEN, dtype=np.int64)
    keep = [_host_ptr(a) for a in (ce_rowptr, ce_col, se_rowptr, se_col)]
    _check(L.mpld_decompose_batch(n_layouts, lo_p, int(n), *[p for p, _ in keep], int(k), float(alpha),
                                  int(max_steps), int(flags), col_p, nc.ctypes.data, ns.ctypes.data,
                                  cost.ctypes.data, stats.ctypes.data))
    return {"colors": colors, "n_conflicts": nc, "n_stitches": ns, "cost": cost,
            "stats": dict(zip(STAT_NAMES, stats.tolist()))}


def decompose_graph(g, k: int, alpha: float, max_steps: int = 0, flags: int = 0):
    """Convenience: host batch call on an object with n, layout_offsets, ce_rowptr,
    ce_col, se_rowptr, se_col attributes (e.g. synth.DecompGraph)."""
    return mpld_decompose_batch(g.layout_offsets, g.n, g.ce_rowptr, g.ce_col, g.se_rowptr, g.se_col, k, alpha,
                                max_steps, flags)


class Context:
    """Device-resident entry point (`mpld_context_*`, `mpld_decompose_device`)."""

    def __init__(self, device: int = 0, max_vertices: int = 1 << 16, max_layouts: int = 16):
        L = lib()
        h = _vp()
        _check(L.mpld_context_create(int(device), int(max_vertices), int(max_layouts), ctypes.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().mpld_context_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def submit(self, layout_offsets, n, ce_rowptr, ce_col, se_rowptr, se_col, k, alpha, max_steps=0, flags=0,
               out=None):
        """C ABI `mpld_decompose_batch_async`: host buffers (numpy arrays or CPU
        tensors; pinned memory for asynchronous copies), returns a ticket.  The
        result dict (colors, n_conflicts, n_stitches, cost, stats) is complete
        after `wait(ticket)`; `out` may supply preallocated output arrays."""
        L = lib()
        lo_p, lo = _host_ptr(layout_offsets)
        n_layouts = int(len(lo) - 1) if not hasattr(lo, "numel") else int(lo.numel() - 1)
        if out is None:
            out = {"colors": np.empty(max(int(n), 0), dtype=np.int32),
                   "n_conflicts": np.zeros(n_layouts, dtype=np.int64),
                   "n_stitches": np.zeros(n_layouts, dtype=np.int64),
                   "cost": np.zeros(n_layouts, dtype=np.float64),
                   "stats": np.zeros(MPLD_STAT_LEN, dtype=np.int64)}
        keep = [lo] + [_host_ptr(a) for a in (ce_rowptr, ce_col, se_rowptr, se_col)]
        ptr = {key: _out_ptr(v, _OUT_DTYPES[key], key) for key, v in out.items()}
        t = ctypes.c_int64()
        _check(L.mpld_decompose_batch_async(self._h, n_layouts, lo_p, int(n), *[p for p, _ in keep[1:]], int(k),
                                            float(alpha), int(max_steps), int(flags), ptr["colors"],
                                            ptr["n_conflicts"], ptr["n_stitches"], ptr["cost"], ptr["stats"],
                                            ctypes.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (keep, out)
        return t.value

    def submit_pairs(self, layout_offsets, n, ce_rowptr, ce_col, stitch_pairs, k, alpha, max_steps=0, flags=0,
                     out=None):
        """C ABI `mpld_decompose_batch_pairs_async`: as `submit`, with the stitch
        edges as an int32 array of (u, v) pairs (shape [m, 2] or flat [2m]),
        each edge once; the SE CSR is built on the device."""
        L = lib()
        lo_p, lo = _host_ptr(layout_offsets)
        n_layouts = int(len(lo) - 1) if not hasattr(lo, "numel") else int(lo.numel() - 1)
        if out is None:
            out = {"colors": np.empty(max(int(n), 0), dtype=np.int32),
                   "n_conflicts": np.zeros(n_layouts, dtype=np.int64),
                   "n_stitches": np.zeros(n_layouts, dtype=np.int64),
                   "cost": np.zeros(n_layouts, dtype=np.float64),
                   "stats": np.zeros(MPLD_STAT_LEN, dtype=np.int64)}
        sp = _host_ptr(stitch_pairs)
        m = int(sp[1].numel() if hasattr(sp[1], "numel") else np.asarray(sp[1]).size) // 2
        keep = [lo] + [_host_ptr(a) for a in (ce_rowptr, ce_col)] + [sp]
        ptr = {key: _out_ptr(v, _OUT_DTYPES[key], key) for key, v in out.items()}
        t = ctypes.c_int64()
        _check(L.mpld_decompose_batch_pairs_async(self._h, n_layouts, lo_p, int(n), keep[1][0], keep[2][0], m, sp[0],
                                                  int(k), float(alpha), int(max_steps), int(flags), ptr["colors"],
                                                  ptr["n_conflicts"], ptr["n_stitches"], ptr["cost"], ptr["stats"],
                                                  ctypes.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (keep, out)
        return t.value

    def submit_upper(self, layout_offsets, n, ce_up_deg, ce_up_col, stitch_pairs, k, alpha, max_steps=0, flags=0,
                     out=None):
        """C ABI `mpld_decompose_batch_upper_async`: as `submit_pairs`, with the
        conflict edges as the upper triangle of their CSR (ce_up_deg: uint8 [n]
        counts of neighbours u > v; ce_up_col: int32 neighbours, rows ascending;
        synth.upper_csr builds both); the symmetric CSR is built on the device."""
        L = lib()
        lo_p, lo = _host_ptr(layout_offsets)
        n_layouts = int(len(lo) - 1) if not hasattr(lo, "numel") else int(lo.numel() - 1)
        if out is None:
            out = {"colors": np.empty(max(int(n), 0), dtype=np.int32),
                   "n_conflicts": np.zeros(n_layouts, dtype=np.int64),
                   "n_stitches": np.zeros(n_layouts, dtype=np.int64),
                   "cost": np.zeros(n_layouts, dtype=np.float64),
                   "stats": np.zeros(MPLD_STAT_LEN, dtype=np.int64)}
        dg = _host_ptr(ce_up_deg, np.uint8, "ce_up_deg")
        cu = _host_ptr(ce_up_col, np.int32, "ce_up_col")
        sp = _host_ptr(stitch_pairs)
        m_ce = int(cu[1].numel() if hasattr(cu[1], "numel") else np.asarray(cu[1]).size)
        m_se = int(sp[1].numel() if hasattr(sp[1], "numel") else np.asarray(sp[1]).size) // 2
        keep = [lo, dg, cu, sp]
        ptr = {key: _out_ptr(v, _OUT_DTYPES[key], key) for key, v in out.items()}
        t = ctypes.c_int64()
        _check(L.mpld_decompose_batch_upper_async(self._h, n_layouts, lo_p, int(n), dg[0], m_ce, cu[0], m_se, sp[0],
                                                  int(k), float(alpha), int(max_steps), int(flags), ptr["colors"],
                                                  ptr["n_conflicts"], ptr["n_stitches"], ptr["cost"], ptr["stats"],
                                                  ctypes.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (keep, out)
        return t.value

    def wait(self, ticket: int):
        """C ABI `mpld_wait`: block until `ticket` completed; returns its result dict."""
        keep, out = self._inflight.pop(ticket)
        _check(lib().mpld_wait(self._h, int(ticket)))
        res = dict(out)
        st = res["stats"]
        res["stats"] = dict(zip(STAT_NAMES, (st.tolist() if hasattr(st, "tolist") else list(st))))
        return res

    def decompose_device(self, layout_offsets, n, ce_rowptr, ce_col, se_rowptr, se_col, k, alpha, max_steps,
                         colors, counts, cost, stats=None, flags: int = 0, stream=None):
        """Enqueue the hot path on `stream` (torch.cuda.Stream or raw handle; None =
        torch's current stream).  All tensors on the device; asynchronous."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(colors.device)
        sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream or 0)
        n_layouts = int(layout_offsets.numel() - 1)
        _check(lib().mpld_decompose_device(self._h, _vp(sh), n_layouts, _dev_ptr(layout_offsets), int(n),
                                           _dev_ptr(ce_rowptr), _dev_ptr(ce_col), _dev_ptr(se_rowptr),
                                           _dev_ptr(se_col), int(k), float(alpha), int(max_steps), int(flags),
                                           _dev_ptr(colors), _dev_ptr(counts, np.int64, "counts"),
                                           _dev_ptr(cost, np.float64, "cost"), _dev_ptr(stats, np.int64, "stats")))

    # ---- phase-split calls for a batch sharded over processes (include/mpld.h) ----
    @staticmethod
    def _stream(stream, like):
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(like.device)
        return _vp(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream or 0))

    def prepare_device(self, layout_offsets, n, ce_rowptr, ce_col, se_rowptr, se_col, k, colors, counts,
                       flags: int = 0, stream=None):
        """Phase 1 (validate?, simplification, components); colours set to -1."""
        _check(lib().mpld_prepare_device(self._h, self._stream(stream, colors), int(layout_offsets.numel() - 1),
                                         _dev_ptr(layout_offsets), int(n), _dev_ptr(ce_rowptr), _dev_ptr(ce_col),
                                         _dev_ptr(se_rowptr), _dev_ptr(se_col), int(k), int(flags),
                                         _dev_ptr(colors), _dev_ptr(counts, np.int64, "counts")))

    def search_device(self, alpha, max_steps, shard_index, shard_count, colors, stream=None):
        """Phase 2: search the components of this shard, colours of the others stay -1."""
        _check(lib().mpld_search_device(self._h, self._stream(stream, colors), float(alpha), int(max_steps),
                                        int(shard_index), int(shard_count), _dev_ptr(colors)))

    def shard_export(self, colors, pairs, count, stream=None):
        """Phase 3 (compact): the (vertex, colour) pairs of this shard's search into
        pairs (int32 [>= 2n]), their number into count (int64 [1]), on the device."""
        if pairs.numel() < 2 * int(colors.numel()):
            raise ValueError("pairs must hold 2 * n int32")
        _check(lib().mpld_shard_export(self._h, self._stream(stream, colors), _dev_ptr(colors), _dev_ptr(pairs),
                                       _dev_ptr(count, np.int64, "count")))

    def shard_import(self, pairs, colors, stream=None):
        """Phase 3 (compact): scatter (vertex, colour) pairs (int32, flat; vertex < 0 = padding) into colors."""
        _check(lib().mpld_shard_import(self._h, self._stream(stream, colors), _dev_ptr(pairs),
                                       int(pairs.numel() // 2), _dev_ptr(colors)))

    def finish_device(self, alpha, colors, counts, cost, stats=None, stream=None):
        """Phase 3: recovery and Eq. (1) (after the colours of all shards are combined)."""
        _check(lib().mpld_finish_device(self._h, self._stream(stream, colors), float(alpha), _dev_ptr(colors),
                                        _dev_ptr(counts, np.int64, "counts"), _dev_ptr(cost, np.float64, "cost"),
                                        _dev_ptr(stats, np.int64, "stats")))

    def set_timing(self, enable: bool):
        _check(lib().mpld_context_set_timing(self._h, 1 if enable else 0))

    def reset_timing(self):
        _check(lib().mpld_context_reset_timing(self._h))

    def debug(self, extra: int = 0):
        """Diagnostics of the last call (include/mpld.h mpld_context_debug); `extra`
        more words: the heavy-search trace of MPLD_DIAG_HEAVY builds."""
        out = np.zeros(96 + int(extra), dtype=np.int64)
        _check(lib().mpld_context_debug(self._h, out.ctypes.data, 96 + int(extra)))
        return out

    def kernel_times(self):
        """{kernel name: (accumulated ms, launches)} since the last reset."""
        L = lib()
        out = {}
        for i in range(L.mpld_kernel_count()):
            ms, cnt = ctypes.c_double(), ctypes.c_int64()
            _check(L.mpld_context_kernel_time(self._h, i, ctypes.byref(ms), ctypes.byref(cnt)))
            out[L.mpld_kernel_name(i).decode()] = (ms.value, cnt.value)
        return out

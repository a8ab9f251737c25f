"""B200-native speculative chunked DFA membership test (arXiv:1210.5093).

Thin ctypes binding of ``libdfa.so`` (C ABI in ``include/dfa.h``).  Function
names are the C names; this module only marshals arguments (numpy arrays for
host memory, torch CUDA tensors or raw ints for device memory, torch streams).
Every step of the path runs in the library's CUDA kernels; there is no CPU
fallback: if ``libdfa.so`` is missing, importing the functions raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

from .build import LIB
from .build import build  # noqa: F401

__all__ = [
    "DfaError", "dfa_create", "dfa_create_ex", "dfa_destroy", "dfa_get_info", "dfa_domain",
    "dfa_set_chunk_ratio", "dfa_plan_bounds", "dfa_match", "dfa_match_host", "dfa_chunk_maps",
    "dfa_chunk_maps_at", "dfa_get_last_device_error", "dfa_set_option", "dfa_get_stats",
    "dfa_status_string", "dfa_error_detail", "dfa_segment_map", "dfa_fold_segments",
    "dfa_lookahead_maps", "dfa_match_batch", "dfa_gather_ceiling", "dfa_segment_chunk_maps", "Dfa", "lib",
    "EXPORTED",
]

DFA_OK, DFA_ERR_ARG, DFA_ERR_STATES, DFA_ERR_ALPHABET, DFA_ERR_CHUNKS = 0, 1, 2, 3, 4
DFA_ERR_SYMBOL, DFA_ERR_OOM, DFA_ERR_CUDA, DFA_ERR_INTERNAL = 5, 6, 7, 8
DFA_CREATE_HOST_ONLY = 1
DFA_CREATE_FULL_DOMAIN = 2
DFA_OPT_SUBCHUNK_TARGET, DFA_OPT_CONVERGENCE, DFA_OPT_PROFILE, DFA_OPT_THREADS_PER_CTA = 1, 2, 3, 4
DFA_OPT_TREE_FANIN = 5
DFA_OPT_FOLD_IN_TREE = 6
DFA_OPT_WARP_COMPOSE = 7
DFA_OPT_GRAPHS = 8
DFA_OPT_MAX_LANES = 9
DFA_OPT_HOST_PIECE = 10
DFA_OPT_EARLY_EXIT = 11
DFA_OPT_STICKY_PARKING = 12
DFA_OPT_COUNT_WORK = 13
DFA_OPT_FUSED_TAIL = 14
DFA_OPT_FACTORED = 15
DFA_OPT_LOOKAHEAD2 = 16
DFA_OPT_TMA_INPUT = 17


def DFA_CREATE_TABLE_MODE(m: int) -> int:
    """dfa_create_ex flag forcing table layout m (a TABLE_MODES key), include/dfa.h."""
    return (int(m) & 0xF) << 8

TABLE_MODES = {1: "ident_u8", 2: "ident_u16", 3: "window_u8", 4: "window_u16", 5: "packed9", 6: "global_u16",
               7: "rep8_u8", 8: "rep4_u8", 9: "ident_u8_pad"}


class DfaInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in (
        "num_states", "alphabet_size", "num_classes", "i_max", "gamma_num", "gamma_den", "num_dead",
        "dead_state", "num_absorbing", "table_mode", "table_bytes", "c_num", "c_den", "device_ready")]


class DfaStats(ctypes.Structure):
    _fields_ = [("input_bytes", ctypes.c_uint64), ("num_subchunks", ctypes.c_uint64),
                ("num_kernels", ctypes.c_uint32),
                ("profiled", ctypes.c_uint32), ("kernel_ms", ctypes.c_float * 8),
                ("kernel_name", (ctypes.c_char * 32) * 8), ("host_bytes", ctypes.c_uint64),
                ("work_lookups", ctypes.c_uint64 * 2), ("work_calls", ctypes.c_uint32)]


class DfaError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        detail = dfa_error_detail() if status in (DFA_ERR_CUDA, DFA_ERR_OOM) else ""
        super().__init__(f"{what}: {dfa_status_string(status)} ({status}) {detail}".rstrip())


# every function declared in include/dfa.h
EXPORTED = ["dfa_create", "dfa_create_ex", "dfa_destroy", "dfa_get_info", "dfa_domain",
            "dfa_set_chunk_ratio", "dfa_plan_bounds", "dfa_match", "dfa_match_host", "dfa_chunk_maps",
            "dfa_chunk_maps_at", "dfa_get_last_device_error", "dfa_set_option", "dfa_get_stats",
            "dfa_status_string", "dfa_error_detail", "dfa_segment_map", "dfa_fold_segments",
            "dfa_lookahead_maps", "dfa_match_batch", "dfa_gather_ceiling", "dfa_segment_chunk_maps"]

_lib = None


def lib():
    """Load libdfa.so; raise if it is missing (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built: run paper_1210_5093_b200.build.build() "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB)
        V, u16, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint16, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        sig = {
            "dfa_create": [V, u32, u32, u16, V, V],
            "dfa_create_ex": [V, u32, u32, u16, V, u32, V],
            "dfa_destroy": [V],
            "dfa_get_info": [V, V],
            "dfa_domain": [V, u32, V, V],
            "dfa_set_chunk_ratio": [V, u32, u32],
            "dfa_plan_bounds": [u64, u32, u32, u32, V],
            "dfa_match": [V, V, u64, V, V, V],
            "dfa_match_host": [V, V, u64, V, V, V],
            "dfa_chunk_maps": [V, V, u64, u32, V, V, V, V, V, V],
            "dfa_chunk_maps_at": [V, V, u64, u32, V, V, V, V, V, V],
            "dfa_get_last_device_error": [V],
            "dfa_set_option": [V, u32, ctypes.c_int64],
            "dfa_get_stats": [V, V],
            "dfa_segment_map": [V, V, u64, ctypes.c_int32, V, V],
            "dfa_fold_segments": [V, V, V, u32, V, V],
            "dfa_lookahead_maps": [V, V, u64, u32, V, V, u32, V, V, V, V],
            "dfa_match_batch": [V, V, u64, V, u32, V, V, V],
            "dfa_gather_ceiling": [V, V, u64, V, V, V, V],
            "dfa_segment_chunk_maps": [V, V, u64, u32, ctypes.c_int32, V, V, V, V, V],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = i32
        L.dfa_status_string.argtypes = [i32]
        L.dfa_status_string.restype = ctypes.c_char_p
        L.dfa_error_detail.argtypes = []
        L.dfa_error_detail.restype = ctypes.c_char_p
        _lib = L
    return _lib


def dfa_error_detail() -> str:
    return lib().dfa_error_detail().decode()


def dfa_status_string(status: int) -> str:
    return lib().dfa_status_string(int(status)).decode()


def _ck(status: int, what: str):
    if status != DFA_OK:
        raise DfaError(status, what)


def _ptr(x) -> Optional[int]:
    """Device/host pointer of a torch tensor, numpy array or int (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# --------------------------------------------------------------------------- calls
def dfa_create_ex(table: np.ndarray, q0: int, accept_bitmap: np.ndarray, flags: int = 0) -> ctypes.c_void_p:
    t = np.ascontiguousarray(table, dtype=np.uint16)
    nq, ns = t.shape
    bm = np.ascontiguousarray(accept_bitmap, dtype=np.uint8)
    if bm.size * 8 < nq:
        raise ValueError("accept bitmap too short")
    h = ctypes.c_void_p()
    _ck(lib().dfa_create_ex(t.ctypes.data, nq, ns, int(q0), bm.ctypes.data, int(flags), ctypes.byref(h)),
        "dfa_create")
    return h


def dfa_create(table: np.ndarray, q0: int, accept_bitmap: np.ndarray) -> ctypes.c_void_p:
    return dfa_create_ex(table, q0, accept_bitmap, 0)


def dfa_destroy(h):
    _ck(lib().dfa_destroy(h), "dfa_destroy")


def dfa_get_info(h) -> dict:
    info = DfaInfo()
    _ck(lib().dfa_get_info(h, ctypes.byref(info)), "dfa_get_info")
    d = {n: getattr(info, n) for n, _ in DfaInfo._fields_}
    d["table_mode_name"] = TABLE_MODES.get(d["table_mode"], "?")
    return d


def dfa_domain(h, sigma: int) -> np.ndarray:
    info = dfa_get_info(h)
    out = np.zeros(max(info["i_max"], 1), np.uint16)
    cnt = ctypes.c_uint32()
    _ck(lib().dfa_domain(h, int(sigma), out.ctypes.data, ctypes.byref(cnt)), "dfa_domain")
    return out[:cnt.value].copy()


def dfa_set_chunk_ratio(h, c_num: int, c_den: int = 1):
    _ck(lib().dfa_set_chunk_ratio(h, int(c_num), int(c_den)), "dfa_set_chunk_ratio")


def dfa_plan_bounds(n: int, P: int, c_num: int, c_den: int = 1) -> np.ndarray:
    out = np.zeros(P + 1, np.uint64)
    _ck(lib().dfa_plan_bounds(int(n), int(P), int(c_num), int(c_den), out.ctypes.data), "dfa_plan_bounds")
    return out


def dfa_match(h, dev_input, n: Optional[int] = None, stream=None) -> Tuple[int, bool]:
    n = dev_input.numel() if n is None else int(n)
    fs = ctypes.c_uint16()
    acc = ctypes.c_int()
    _ck(lib().dfa_match(h, _ptr(dev_input), n, _stream(stream), ctypes.byref(fs), ctypes.byref(acc)),
        "dfa_match")
    return fs.value, bool(acc.value)


def dfa_match_host(h, host_input, n: Optional[int] = None, stream=None) -> Tuple[int, bool]:
    if isinstance(host_input, np.ndarray):
        n = host_input.size if n is None else int(n)
    else:
        n = host_input.numel() if n is None else int(n)
    fs = ctypes.c_uint16()
    acc = ctypes.c_int()
    _ck(lib().dfa_match_host(h, _ptr(host_input), n, _stream(stream), ctypes.byref(fs), ctypes.byref(acc)),
        "dfa_match_host")
    return fs.value, bool(acc.value)


def dfa_chunk_maps(h, dev_input, P: int, dev_bounds, dev_chunk0_end, dev_maps, dev_chunk_start=None,
                   dev_final=None, n: Optional[int] = None, stream=None):
    n = dev_input.numel() if n is None else int(n)
    _ck(lib().dfa_chunk_maps(h, _ptr(dev_input), n, int(P), _stream(stream), _ptr(dev_bounds),
                             _ptr(dev_chunk0_end), _ptr(dev_maps), _ptr(dev_chunk_start), _ptr(dev_final)),
        "dfa_chunk_maps")


def dfa_chunk_maps_at(h, dev_input, P: int, dev_bounds_in, dev_chunk0_end, dev_maps, dev_chunk_start=None,
                      dev_final=None, n: Optional[int] = None, stream=None):
    n = dev_input.numel() if n is None else int(n)
    _ck(lib().dfa_chunk_maps_at(h, _ptr(dev_input), n, int(P), _ptr(dev_bounds_in), _stream(stream),
                                _ptr(dev_chunk0_end), _ptr(dev_maps), _ptr(dev_chunk_start), _ptr(dev_final)),
        "dfa_chunk_maps_at")


def dfa_lookahead_maps(h, dev_input, P: int, dev_bounds, dev_maps, r: int, dev_domains, dev_domain_sizes,
                       dev_maps_r, n: Optional[int] = None, stream=None):
    """Chunk maps restricted to r reverse lookahead symbols (Eq.istatesm)."""
    n = dev_input.numel() if n is None else int(n)
    _ck(lib().dfa_lookahead_maps(h, _ptr(dev_input), n, int(P), _ptr(dev_bounds), _ptr(dev_maps), int(r),
                                 _stream(stream), _ptr(dev_domains), _ptr(dev_domain_sizes), _ptr(dev_maps_r)),
        "dfa_lookahead_maps")


def dfa_match_batch(h, dev_data, dev_offsets, dev_final, dev_accept, data_len: Optional[int] = None, stream=None):
    """Independent inputs dev_data[off[j]:off[j+1]] (dev_offsets: device uint64/int64 tensor of
    count+1 entries) matched from q0; finals -> dev_final (uint16), accept -> dev_accept (uint8)."""
    n = dev_data.numel() if data_len is None else int(data_len)
    count = dev_offsets.numel() - 1
    _ck(lib().dfa_match_batch(h, _ptr(dev_data), n, _ptr(dev_offsets), int(count), _stream(stream),
                              _ptr(dev_final), _ptr(dev_accept)), "dfa_match_batch")


def dfa_segment_map(h, dev_input, lookahead: int, dev_row, n: Optional[int] = None, stream=None):
    """Map of one input segment over I_sigma(lookahead) (lookahead -1: from q0)."""
    n = dev_input.numel() if n is None else int(n)
    _ck(lib().dfa_segment_map(h, _ptr(dev_input), n, int(lookahead), _stream(stream), _ptr(dev_row)),
        "dfa_segment_map")


def dfa_segment_chunk_maps(h, dev_input, P: int, lookahead: int, dev_bounds, dev_chunk0_row, dev_maps,
                           dev_segment_row, n: Optional[int] = None, stream=None):
    """Per-GPU step of the sharded path (include/dfa.h): P chunks of the segment, chunk 0
    from {q0} (lookahead -1) or I_sigma(lookahead); writes bounds, chunk 0's row, the maps of
    chunks 1.. and the segment's composed map row."""
    n = dev_input.numel() if n is None else int(n)
    _ck(lib().dfa_segment_chunk_maps(h, _ptr(dev_input), n, P, int(lookahead), _stream(stream), _ptr(dev_bounds),
                                     _ptr(dev_chunk0_row), _ptr(dev_maps), _ptr(dev_segment_row)),
        "dfa_segment_chunk_maps")


def dfa_gather_ceiling(h, dev_input=None, dev_out=None, stream=None, length=None):
    """Measurement aid (include/dfa.h): run the match step alone, one lane per thread
    from q0.  Returns (threads, bytes_per_thread); with dev_out None only queries them."""
    per = ctypes.c_uint64(0)
    nt = ctypes.c_uint32(0)
    n = int(length if length is not None else (dev_input.numel() if dev_input is not None else 0))
    _ck(lib().dfa_gather_ceiling(h, _ptr(dev_input) if dev_input is not None else None, n, _stream(stream),
                                 _ptr(dev_out) if dev_out is not None else None, ctypes.byref(per),
                                 ctypes.byref(nt)), "dfa_gather_ceiling")
    return int(nt.value), int(per.value)


def dfa_fold_segments(h, dev_rows, dev_lookahead, G: int, dev_final, stream=None):
    _ck(lib().dfa_fold_segments(h, _ptr(dev_rows), _ptr(dev_lookahead), int(G), _stream(stream), _ptr(dev_final)),
        "dfa_fold_segments")


def dfa_get_last_device_error(h) -> int:
    return int(lib().dfa_get_last_device_error(h))


def dfa_set_option(h, key: int, value: int):
    _ck(lib().dfa_set_option(h, int(key), int(value)), "dfa_set_option")


def dfa_get_stats(h) -> dict:
    """Last-call counters, plus per-section kernel milliseconds summed over the
    calls since the previous dfa_get_stats (DFA_OPT_PROFILE)."""
    s = DfaStats()
    _ck(lib().dfa_get_stats(h, ctypes.byref(s)), "dfa_get_stats")
    d = {"input_bytes": s.input_bytes, "num_subchunks": s.num_subchunks,
         "num_kernels": s.num_kernels, "profiled_calls": s.profiled, "host_bytes": s.host_bytes}
    if s.profiled:
        d["kernel_ms"] = {bytes(s.kernel_name[i]).split(b"\0")[0].decode(): s.kernel_ms[i]
                          for i in range(8) if s.kernel_name[i][0]}
    if s.work_calls:
        d["work"] = {"converge": int(s.work_lookups[0]), "lanes": int(s.work_lookups[1]), "calls": int(s.work_calls)}
    return d


class Dfa:
    """RAII wrapper: ``with Dfa(table, q0, bitmap) as d: d.match(x)``."""

    def __init__(self, table, q0, accept_bitmap, flags: int = 0):
        self.h = dfa_create_ex(table, q0, accept_bitmap, flags)
        self.info = dfa_get_info(self.h)

    def close(self):
        if self.h is not None:
            dfa_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def match(self, dev_input, stream=None):
        return dfa_match(self.h, dev_input, stream=stream)

    def domain(self, sigma: int):
        return dfa_domain(self.h, sigma)

    def chunk_maps(self, dev_input, P: int, with_starts: bool = False, stream=None):
        """Allocate outputs with torch and return (bounds, e0, maps, starts, final) as torch tensors."""
        import torch
        dev = dev_input.device
        imax = self.info["i_max"]
        bounds = torch.empty(P + 1, dtype=torch.int64, device=dev)
        e0 = torch.empty(1, dtype=torch.int16, device=dev)
        maps = torch.empty(max(P - 1, 1) * imax, dtype=torch.int16, device=dev)
        starts = torch.empty(P, dtype=torch.int16, device=dev) if with_starts else None
        final = torch.empty(2, dtype=torch.int16, device=dev)
        dfa_chunk_maps(self.h, dev_input, P, bounds, e0, maps, starts, final, stream=stream)
        return bounds, e0, maps.view(max(P - 1, 1), imax)[:P - 1], starts, final

    def lookahead_maps(self, dev_input, bounds, maps, r: int, stream=None):
        """Restrict chunk_maps() results to r reverse lookahead symbols; returns
        (domains, sizes, maps_r) as torch tensors ([P-1, i_max], [P-1], [P-1, i_max])."""
        import torch
        dev = dev_input.device
        P = bounds.numel() - 1
        imax = self.info["i_max"]
        doms = torch.empty(max(P - 1, 1) * imax, dtype=torch.int16, device=dev)
        sizes = torch.empty(max(P - 1, 1), dtype=torch.int16, device=dev)
        maps_r = torch.empty(max(P - 1, 1) * imax, dtype=torch.int16, device=dev)
        dfa_lookahead_maps(self.h, dev_input, P, bounds, maps, r, doms, sizes, maps_r, stream=stream)
        return doms.view(max(P - 1, 1), imax)[:P - 1], sizes[:P - 1], maps_r.view(max(P - 1, 1), imax)[:P - 1]

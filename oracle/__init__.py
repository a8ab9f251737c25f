"""CPU oracle for the speculative chunked DFA membership test (arXiv:1210.5093).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this package.  It shares no code with the CUDA product path
(``paper_1210_5093_b200``): the arithmetic lives in ``oracle.c`` (plain C,
fp-free, every function citing the PAPER.md passage it writes out) and this
module only marshals numpy arrays into it.

Parity status: every function below is pinned
by ``tests/test_oracle_pins.py`` against worked values printed in the paper,
brute-force search, closed forms or invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, BAD_SYMBOL, BAD_ARG, NOT_IN_DOMAIN = 0, 1, 2, 3


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C11, -O2) into liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-pthread", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u16, u32, u64 = ctypes.c_uint16, ctypes.c_uint32, ctypes.c_uint64
        L.oracle_run.argtypes = [P, u32, u32, u16, P, u64, P]
        L.oracle_run_record.argtypes = [P, u32, u32, u16, P, u64, P, u32, P, P]
        L.oracle_accepts.argtypes = [P, u16]
        L.oracle_error_states.argtypes = [P, u32, u32, P, P]
        L.oracle_error_states.restype = u32
        L.oracle_initial_states.argtypes = [P, u32, u32, P, u32, P]
        L.oracle_initial_states.restype = u32
        L.oracle_initial_states_r.argtypes = [P, u32, u32, P, P, u32, P]
        L.oracle_initial_states_r.restype = u32
        L.oracle_chunk_map_r.argtypes = [P, u32, u32, P, P, u64, u64, u64, u32, u32, P, P, P]
        L.oracle_imax.argtypes = [P, u32, u32, P]
        L.oracle_imax.restype = u32
        L.oracle_chunk_bounds.argtypes = [u64, u32, u32, P, P]
        L.oracle_chunk_map.argtypes = [P, u32, u32, P, P, u64, u64, u64, u32, P, P]
        L.oracle_maps.argtypes = [P, u32, u32, P, u16, P, u64, P, u32, u32, u32, P, P]
        L.oracle_fold.argtypes = [P, u32, u32, P, P, P, u32, u32, u16, P, P]
        L.oracle_compose_dense.argtypes = [P, P, u32, P]
        for f in ("oracle_run", "oracle_run_record", "oracle_chunk_bounds",
                  "oracle_chunk_map", "oracle_maps", "oracle_fold", "oracle_accepts"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(st: int, what: str):
    if st != OK:
        raise OracleError(f"{what}: oracle status {st}")


class Dfa:
    """A DFA (Q, Sigma, delta, q0, F) as in P:149-163, table[q, c] = delta(q, c)."""

    def __init__(self, table, q0: int, accepting: Sequence[int] | np.ndarray):
        self.table = np.ascontiguousarray(np.asarray(table, dtype=np.uint16))
        assert self.table.ndim == 2
        self.nq, self.ns = self.table.shape
        self.q0 = int(q0)
        acc = np.zeros(self.nq, dtype=bool)
        acc_in = np.asarray(accepting)
        if acc_in.dtype == bool:
            acc[:] = acc_in
        else:
            acc[np.asarray(acc_in, dtype=np.int64)] = True
        self.accepting = acc
        self.accept_bitmap = np.packbits(acc, bitorder="little")
        if self.accept_bitmap.size == 0:
            self.accept_bitmap = np.zeros(1, np.uint8)
        self._dead = None

    # Alg.seqmatch
    def run(self, x: np.ndarray) -> int:
        x = np.ascontiguousarray(x, dtype=np.uint8)
        out = np.zeros(1, np.uint16)
        _check(lib().oracle_run(_p(self.table), self.nq, self.ns, self.q0, _p(x), x.size, _p(out)),
               "oracle_run")
        return int(out[0])

    # Alg.seqmatch lines 4-6: accept iff the final state is in F
    def accepts(self, x: np.ndarray) -> bool:
        return bool(lib().oracle_accepts(_p(self.accept_bitmap), self.run(x)))

    def run_record(self, x: np.ndarray, positions: np.ndarray):
        x = np.ascontiguousarray(x, dtype=np.uint8)
        pos = np.ascontiguousarray(positions, dtype=np.uint64)
        at = np.zeros(max(pos.size, 1), np.uint16)
        out = np.zeros(1, np.uint16)
        _check(lib().oracle_run_record(_p(self.table), self.nq, self.ns, self.q0, _p(x), x.size,
                                       _p(pos), pos.size, _p(at), _p(out)), "oracle_run_record")
        return at[:pos.size].copy(), int(out[0])

    @property
    def dead(self) -> np.ndarray:
        """Error states Z (reading R1)."""
        if self._dead is None:
            d = np.zeros(self.nq, np.uint8)
            lib().oracle_error_states(_p(self.table), self.nq, self.ns, _p(self.accept_bitmap), _p(d))
            self._dead = d
        return self._dead

    def initial_states(self, sigma: int) -> np.ndarray:
        """I_sigma, Eq.istates / Alg.MatchingInitialStates l.1-7."""
        out = np.zeros(max(self.nq, 1), np.uint16)
        c = lib().oracle_initial_states(_p(self.table), self.nq, self.ns, _p(self.dead), int(sigma),
                                        _p(out))
        return out[:c].copy()

    def initial_states_r(self, syms: Sequence[int]) -> np.ndarray:
        """I_{s1..sr}, Eq.istatesm / Alg.TwoSymISet (symbols in matching order)."""
        s = np.ascontiguousarray(np.asarray(syms, dtype=np.uint8))
        out = np.zeros(max(self.nq, 1), np.uint16)
        c = lib().oracle_initial_states_r(_p(self.table), self.nq, self.ns, _p(self.dead), _p(s),
                                          s.size, _p(out))
        return out[:c].copy()

    def imax(self) -> int:
        """Eq.MaxIstates."""
        return int(lib().oracle_imax(_p(self.table), self.nq, self.ns, _p(self.dead)))

    def chunk_map(self, x: np.ndarray, begin: int, end: int, row_len: int):
        x = np.ascontiguousarray(x, dtype=np.uint8)
        row = np.zeros(max(row_len, 1), np.uint16)
        cnt = np.zeros(1, np.uint32)
        _check(lib().oracle_chunk_map(_p(self.table), self.nq, self.ns, _p(self.dead), _p(x), x.size,
                                      int(begin), int(end), row_len, _p(row), _p(cnt)),
               "oracle_chunk_map")
        return row[:row_len].copy(), int(cnt[0])

    def chunk_map_r(self, x: np.ndarray, begin: int, end: int, r: int, row_len: int):
        """(domain, row, |domain|) of chunk [begin, end) over I_{s1..sL}, L = min(r, begin)
        lookahead symbols (Eq.istatesm)."""
        x = np.ascontiguousarray(x, dtype=np.uint8)
        row = np.zeros(max(row_len, 1), np.uint16)
        dom = np.zeros(max(row_len, 1), np.uint16)
        cnt = np.zeros(1, np.uint32)
        _check(lib().oracle_chunk_map_r(_p(self.table), self.nq, self.ns, _p(self.dead), _p(x), x.size,
                                        int(begin), int(end), int(r), row_len, _p(dom), _p(row), _p(cnt)),
               "oracle_chunk_map_r")
        return dom[:row_len].copy(), row[:row_len].copy(), int(cnt[0])

    def maps(self, x: np.ndarray, bounds: np.ndarray, row_len: int, threads: int = 0):
        """(chunk0_end, maps[(P-1), row_len]) for the partition `bounds` (P+1 entries)."""
        x = np.ascontiguousarray(x, dtype=np.uint8)
        b = np.ascontiguousarray(bounds, dtype=np.uint64)
        P = b.size - 1
        maps = np.zeros((max(P - 1, 1), max(row_len, 1)), np.uint16)
        e0 = np.zeros(1, np.uint16)
        threads = threads or (os.cpu_count() or 1)
        _check(lib().oracle_maps(_p(self.table), self.nq, self.ns, _p(self.dead), self.q0, _p(x),
                                 x.size, _p(b), P, row_len, threads, _p(e0), _p(maps)), "oracle_maps")
        return int(e0[0]), maps[:P - 1, :row_len].copy()

    def fold(self, x: np.ndarray, bounds: np.ndarray, row_len: int, chunk0_end: int,
             maps: np.ndarray) -> int:
        """Eq.SeqReduction."""
        x = np.ascontiguousarray(x, dtype=np.uint8)
        b = np.ascontiguousarray(bounds, dtype=np.uint64)
        m = np.ascontiguousarray(maps, dtype=np.uint16)
        if m.size == 0:
            m = np.zeros(1, np.uint16)
        out = np.zeros(1, np.uint16)
        _check(lib().oracle_fold(_p(self.table), self.nq, self.ns, _p(self.dead), _p(x), _p(b),
                                 b.size - 1, row_len, int(chunk0_end), _p(m), _p(out)), "oracle_fold")
        return int(out[0])


def chunk_bounds(n: int, P: int, m: int, capacities: Optional[Sequence[int]] = None) -> np.ndarray:
    """Eq.Weights + Eq.LZero + Eq.StartPosition/EndPosition; returns P+1 half-open bounds."""
    cap = np.ascontiguousarray(np.ones(P, np.uint64) if capacities is None
                               else np.asarray(capacities, dtype=np.uint64))
    out = np.zeros(P + 1, np.uint64)
    _check(lib().oracle_chunk_bounds(int(n), int(P), int(m), _p(cap), _p(out)), "oracle_chunk_bounds")
    return out


def chunk_bounds_ratio(n: int, P: int, c_num: int, c_den: int) -> np.ndarray:
    """Bounds for a chunk-0 length ratio c = c_num/c_den (homogeneous chunks 1..P-1).

    Chosen as capacities M_0 = c_num, M_i = c_den (i >= 1) with m = 1 states to
    match, so that w_0*m/w_i = c (Eq.LZero); reading R3.
    """
    caps = np.full(P, c_den, np.uint64)
    caps[0] = c_num
    return chunk_bounds(n, P, 1, caps)


def compose_dense(Li: np.ndarray, Lj: np.ndarray) -> np.ndarray:
    """Eq.MapReduction on dense maps."""
    Li = np.ascontiguousarray(Li, dtype=np.uint16)
    Lj = np.ascontiguousarray(Lj, dtype=np.uint16)
    out = np.zeros_like(Li)
    lib().oracle_compose_dense(_p(Li), _p(Lj), Li.size, _p(out))
    return out

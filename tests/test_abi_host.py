"""CPU-only checks of the C-ABI library (-m "not gpu"): it loads, exports every
symbol include/dfa.h declares, and its host preprocessing (I_sigma, I_max,
gamma, error states, partition formula) agrees with the oracle.  No compute
calls: handles are created host-only."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_1210_5093_b200 as D
import workloads as W
from workloads import automata

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    D.build()
    D.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "dfa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dfa_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 14
    assert sorted(D.EXPORTED) == names
    L = ctypes.CDLL(D.LIB)
    for n in names:
        assert hasattr(L, n), n


def test_binding_constants_match_header():
    """Every DFA_OPT_* / DFA_ERR_* / DFA_CREATE_* value of include/dfa.h has the same value in the binding."""
    src = open(os.path.join(ROOT, "include", "dfa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    consts = dict(re.findall(r"\b(DFA_(?:OPT|ERR|CREATE)_[A-Z0-9_]+)\s*=\s*(\d+)", src))
    assert len([k for k in consts if k.startswith("DFA_OPT_")]) >= 17
    for k, v in consts.items():
        assert getattr(D, k) == int(v), k


def test_plan_division_magic_is_exact():
    """The device's 32-bit sub-chunk arithmetic (kernels.cu udiv_magic / split_range, magics from
    kernels.cuh plan_magic): umulhi(n, floor(2^32 / d)) is floor(n / d) or one less, so one
    correction is exact; and floor(len j / m) = q j + floor(r j / m) with len = q m + r."""
    rng = np.random.default_rng(5)
    ds = [1, 2, 3, 5, 7, 22, 23, 27, 37, 640, 65535, 65536, 65537, (1 << 31) - 1, 1 << 31, (1 << 32) - 1]
    ds += [int(v) for v in rng.integers(1, 1 << 32, 200)]
    for d in ds:
        magic = 0xFFFFFFFF if d <= 1 else (1 << 32) // d
        ns = [0, 1, d - 1, d, d + 1, 2 * d - 1, (1 << 32) - 1, (1 << 32) - d] + [int(v) for v in rng.integers(0, 1 << 32, 50)]
        for n in ns:
            n &= 0xFFFFFFFF
            q = (n * magic) >> 32
            assert n // d - 1 <= q <= n // d
            if n - q * d >= d:
                q += 1
            assert q == n // d, (n, d)
    for _ in range(2000):
        m = int(rng.integers(1, 65537))
        ln = int(rng.integers(0, 1 << 32))
        j = int(rng.integers(0, m + 1))
        q, r = divmod(ln, m)
        assert r * j < (1 << 32) and ln * j // m == q * j + (r * j) // m


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", D.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def host_handle(a):
    return D.dfa_create_ex(a.table, a.q0, a.accept_bitmap, D.DFA_CREATE_HOST_ONLY)


CASES = [
    ("tiny", lambda: W.get("tiny").automaton),
    ("random", lambda: W.get("random").automaton),
    ("keyword", lambda: W.get("keyword").automaton),
    ("protein", lambda: W.get("protein").automaton),
    ("worst", lambda: W.get("worst").automaton),
    ("sink", lambda: automata.random_dfa_with_sink(30, 5, 1)),
    ("sink256", lambda: automata.random_dfa_with_sink(40, 256, 2, 0.6)),
    ("counter", lambda: automata.counter_dfa(9, 7)),
    ("identity", lambda: automata.identity_dfa(5, 3)),
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_host_analysis_matches_oracle(name, make):
    a = make()
    h = host_handle(a)
    try:
        info = D.dfa_get_info(h)
        od = oracle.Dfa(a.table, a.q0, a.accepting)
        assert info["num_states"] == a.nq and info["alphabet_size"] == a.ns
        assert info["device_ready"] == 0
        assert info["i_max"] == max(1, od.imax())
        assert info["num_dead"] == int(od.dead.sum())
        live = a.nq - int(od.dead.sum())
        assert info["gamma_num"] * live == od.imax() * info["gamma_den"]
        for s in range(a.ns):
            assert D.dfa_domain(h, s).tolist() == od.initial_states(s).tolist(), s
        with pytest.raises(D.DfaError):
            if a.ns < 256:
                D.dfa_domain(h, a.ns)
            else:
                raise D.DfaError(5)
    finally:
        D.dfa_destroy(h)


def test_plan_bounds_vs_oracle_formula():
    rng = np.random.default_rng(3)
    for _ in range(500):
        P = int(rng.integers(1, 3000))
        a, b = int(rng.integers(1, 300)), int(rng.integers(1, 50))
        n = int(rng.integers((a + b * (P - 1) + b - 1) // b, 1 << 36))
        assert D.dfa_plan_bounds(n, P, a, b).tolist() == oracle.chunk_bounds_ratio(n, P, a, b).tolist()
    # the paper's worked partitions (Tab.ExampleChunkComp c=8, Fig.InputString c=I_max=2)
    assert D.dfa_plan_bounds(36, 3, 8).tolist() == [0, 28, 32, 36]
    assert D.dfa_plan_bounds(36, 3, 2).tolist() == [0, 18, 27, 36]
    assert D.dfa_plan_bounds(36, 3, 4).tolist() == [0, 24, 30, 36]


def test_plan_bounds_rejects_empty_chunks():
    with pytest.raises(D.DfaError) as e:
        D.dfa_plan_bounds(5, 5, 2)  # n < c + P - 1
    assert e.value.status == D.DFA_ERR_CHUNKS
    assert D.dfa_plan_bounds(6, 5, 2).tolist() == [0, 2, 3, 4, 5, 6]


def test_create_validation():
    t = np.zeros((3, 4), np.uint16)
    bm = np.zeros(1, np.uint8)
    with pytest.raises(D.DfaError) as e:
        D.dfa_create_ex(t, 3, bm, D.DFA_CREATE_HOST_ONLY)
    assert e.value.status == D.DFA_ERR_STATES
    t[1, 2] = 3
    with pytest.raises(D.DfaError) as e:
        D.dfa_create_ex(t, 0, bm, D.DFA_CREATE_HOST_ONLY)
    assert e.value.status == D.DFA_ERR_STATES
    with pytest.raises(D.DfaError) as e:
        D.dfa_create_ex(np.zeros((2, 0), np.uint16).reshape(2, 0), 0, bm, D.DFA_CREATE_HOST_ONLY)
    assert e.value.status == D.DFA_ERR_ALPHABET


def test_host_only_handle_refuses_compute():
    a = W.get("tiny").automaton
    h = host_handle(a)
    try:
        with pytest.raises(D.DfaError) as e:
            D.dfa_match(h, 0, n=10, stream=0)
        assert e.value.status == D.DFA_ERR_ARG
    finally:
        D.dfa_destroy(h)


@pytest.mark.parametrize("name,make,mode", [
    ("tiny", lambda: W.get("tiny").automaton, "ident_u8_pad"),          # < 32 states: one padded copy
    ("random", lambda: W.get("random").automaton, "rep8_u8"),           # 64 states: 8 bank-group copies
    ("keyword", lambda: W.get("keyword").automaton, "ident_u8_pad"),    # 217 states: too big for 8 copies
    ("protein", lambda: W.get("protein").automaton, "window_u16"),      # 342 states, residue window
    ("worst", lambda: W.get("worst").automaton, "packed9"),             # 512 states x 256 columns
    ("sink256", lambda: automata.random_dfa_with_sink(40, 256, 2, 0.6), "rep8_u8"),
    ("poison", lambda: automata.random_dfa(109, 20, 3), "rep8_u8"),     # 109 + poison = 110 states
    ("poison111", lambda: automata.random_dfa(110, 20, 3), "ident_u8_pad"),
])
def test_table_layout_choice(name, make, mode):
    """Host-side layout selection: replicated copies while
    8 x |Q'| x 256 bytes fit the 223 KiB lanes-kernel budget and |Q'| >= 32, else
    padded rows up to 252 states, then the window / packed / global layouts."""
    h = host_handle(make())
    try:
        info = D.dfa_get_info(h)
        assert D.TABLE_MODES[info["table_mode"]] == mode, (name, D.TABLE_MODES[info["table_mode"]])
    finally:
        D.dfa_destroy(h)

"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle,
element by element, on the same seeded inputs.  Bit-exact: every value here is
an integer (state ids, offsets, accept bits)."""
import numpy as np
import pytest

import oracle
import workloads as W
from workloads import automata, inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1210_5093_b200 as D  # noqa: E402

DEV = "cuda:0"


def u16(t):
    return t.cpu().numpy().view(np.uint16)


class Case:
    def __init__(self, aut, x, name=""):
        self.a = aut
        self.x = np.ascontiguousarray(x, dtype=np.uint8)
        self.od = oracle.Dfa(aut.table, aut.q0, aut.accepting)
        self.name = name

    def handle(self, opts=None, flags=0):
        d = D.Dfa(self.a.table, self.a.q0, self.a.accept_bitmap, flags)
        for k, v in (opts or {}).items():
            D.dfa_set_option(d.h, k, v)
        return d


def check_chunk_maps(c: Case, P: int, c_num=1, c_den=1, opts=None, dev=None, maps_rows=None, flags=0):
    """Full parity of bounds, e0, every map entry, true chunk starts, final, accept."""
    d = c.handle(opts, flags)
    try:
        D.dfa_set_chunk_ratio(d.h, c_num, c_den)
        x = c.x
        dx = dev if dev is not None else torch.from_numpy(x).to(DEV)
        bounds, e0, maps, starts, final = d.chunk_maps(dx, P, with_starts=True)
        torch.cuda.synchronize()
        assert D.dfa_get_last_device_error(d.h) == 0
        ob = oracle.chunk_bounds_ratio(x.size, P, c_num, c_den)
        assert np.array_equal(bounds.cpu().numpy().astype(np.uint64), ob), "bounds"
        imax = d.info["i_max"]
        ost, ofin = c.od.run_record(x, ob[:-1])
        assert u16(final)[0] == ofin and u16(final)[1] == int(c.a.accepting[ofin]), "final/accept"
        assert np.array_equal(u16(starts), ost), "chunk starts"
        gm = u16(maps)
        if maps_rows is None:
            oe0, omaps = c.od.maps(x, ob, imax)
            assert u16(e0)[0] == oe0, "e0"
            if P > 1:
                bad = np.argwhere(gm != omaps)
                assert bad.size == 0, f"{len(bad)} map entries differ, first {bad[:3].tolist()}"
        else:  # sampled rows at full size
            for k in maps_rows:
                row, _ = c.od.chunk_map(x, int(ob[k]), int(ob[k + 1]), imax)
                assert np.array_equal(gm[k - 1], row), f"map row {k}"
        return d.info
    finally:
        d.close()


def check_match(c: Case, opts=None, flags=0):
    d = c.handle(opts, flags)
    try:
        fin, acc = d.match(torch.from_numpy(c.x).to(DEV))
        ofin = c.od.run(c.x)
        assert (fin, acc) == (ofin, bool(c.a.accepting[ofin]))
    finally:
        d.close()


# ------------------------------------------------------------------ the five configs (small sizes)
@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_config_small_full_parity(name):
    w = W.get(name)
    x = w.input(w.small_n)
    c = Case(w.automaton, x, name)
    P = min(w.chunks, max(1, x.size // 64))
    check_chunk_maps(c, P)
    check_match(c)


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_config_small_convergence_off(name):
    w = W.get(name)
    x = w.input(min(w.small_n, 1 << 20))
    c = Case(w.automaton, x, name)
    check_chunk_maps(c, 257, opts={D.DFA_OPT_CONVERGENCE: 0})


def test_tiny_hard():
    """P = 65,536 chunks of 16 symbols over the 1 MiB Tiny input (c = 1)."""
    w = W.get("tiny")
    c = Case(w.automaton, w.input(), "tiny-hard")
    check_chunk_maps(c, 65536)


@pytest.mark.parametrize("cn,cd", [(1, 1), (3, 1), (7, 2), (240, 1)])
def test_chunk_ratio_c(cn, cd):
    w = W.get("random")
    c = Case(w.automaton, w.input(1 << 20), "random")
    check_chunk_maps(c, 300, cn, cd)


@pytest.mark.parametrize("target", [1, 7, 1000, 1 << 22])
def test_subchunk_targets(target):
    """The internal execution split must not change any result."""
    w = W.get("keyword")
    c = Case(w.automaton, w.input(1 << 20), "keyword")
    check_chunk_maps(c, 129, opts={D.DFA_OPT_SUBCHUNK_TARGET: target})
    w = W.get("worst")
    c = Case(w.automaton, w.input(1 << 18), "worst")
    check_chunk_maps(c, 33, opts={D.DFA_OPT_SUBCHUNK_TARGET: target})


# ------------------------------------------------------------------ closed forms, special DFAs
def test_counter_dfa_no_convergence():
    a = automata.counter_dfa(37)
    x = inputs.uniform_bytes(3 << 20, seed=4)
    c = Case(a, x, "counter")
    check_chunk_maps(c, 1000)
    check_match(c)
    d = c.handle()
    fin, _ = d.match(torch.from_numpy(x).to(DEV))
    assert fin == int(x.astype(np.int64).sum()) % 37
    d.close()


def test_reset_identity_permutation():
    rng = np.random.default_rng(2)
    f = rng.integers(0, 50, 256)
    for a in (automata.reset_dfa(50, f), automata.identity_dfa(11),
              automata.permutation_dfa(300, 256, 1), automata.permutation_dfa(20, 256, 2)):
        x = inputs.uniform_bytes(1 << 19, seed=5)
        c = Case(a, x, a.name)
        check_chunk_maps(c, 77)
        check_match(c)


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_random_dfas(seed):
    rng = np.random.default_rng(100 + seed)
    nq = int(rng.choice([2, 5, 17, 64, 200, 255, 256, 257, 400, 511, 700, 1500]))
    ns = int(rng.choice([1, 2, 4, 20, 100, 255, 256]))
    kind = seed % 3
    if kind == 0:
        a = automata.random_dfa(nq, ns, seed)
    elif kind == 1:
        a = automata.random_dfa_with_sink(max(nq, 3), ns, seed, float(rng.uniform(0.05, 0.9)))
    else:
        a = automata.random_structured(max(nq, 8), ns, int(rng.integers(1, min(max(nq, 8), 300))),
                                       max(1, nq // 4), seed)
    n = int(rng.integers(1, 1 << 19))
    x = rng.integers(0, ns, n).astype(np.uint8)
    c = Case(a, x, f"fuzz{seed}")
    P = int(rng.integers(1, max(2, min(n, 3000))))
    check_chunk_maps(c, P)
    check_match(c)


@pytest.mark.parametrize("seed", range(6))
def test_arbitrary_partitions(seed):
    """Fold invariant for any partition (dfa_chunk_maps_at), incl. very uneven ones."""
    rng = np.random.default_rng(seed)
    w = W.get(["random", "keyword", "protein", "worst", "tiny", "random"][seed])
    n = 1 << 17
    x = w.input(n)
    c = Case(w.automaton, x, w.name)
    P = int(rng.integers(2, 400))
    cuts = np.sort(rng.choice(np.arange(1, n), P - 1, replace=False))
    if seed % 2:
        cuts = np.unique(np.concatenate([cuts[:P // 2], np.arange(1, min(P // 2, 50) + 1)]))
        P = cuts.size + 1
    ob = np.concatenate([[0], cuts, [n]]).astype(np.uint64)
    d = c.handle()
    try:
        imax = d.info["i_max"]
        dx = torch.from_numpy(x).to(DEV)
        db = torch.from_numpy(ob.astype(np.int64)).to(DEV)
        e0 = torch.empty(1, dtype=torch.int16, device=DEV)
        maps = torch.empty(max(P - 1, 1) * imax, dtype=torch.int16, device=DEV)
        starts = torch.empty(P, dtype=torch.int16, device=DEV)
        final = torch.empty(2, dtype=torch.int16, device=DEV)
        D.dfa_chunk_maps_at(d.h, dx, P, db, e0, maps, starts, final)
        torch.cuda.synchronize()
        oe0, omaps = c.od.maps(x, ob, imax)
        ost, ofin = c.od.run_record(x, ob[:-1])
        assert u16(e0)[0] == oe0
        assert np.array_equal(u16(maps).reshape(-1, imax)[:P - 1], omaps)
        assert np.array_equal(u16(starts), ost)
        assert u16(final)[0] == ofin
    finally:
        d.close()


# ------------------------------------------------------------------ edge cases
def test_edge_lengths_and_chunk_counts():
    a = W.get("keyword").automaton
    for n in (1, 2, 15, 16, 17, 31, 33, 255, 4097):
        x = W.get("keyword").input(n)
        c = Case(a, x)
        check_match(c)
        check_chunk_maps(c, 1)
        check_chunk_maps(c, n)              # n == c + P - 1 with c = 1: every chunk one byte
        if n >= 3:
            check_chunk_maps(c, n - 2, 3, 1)


def test_empty_input_and_errors():
    a = W.get("tiny").automaton
    d = D.Dfa(a.table, a.q0, a.accept_bitmap)
    try:
        empty = torch.empty(0, dtype=torch.uint8, device=DEV)
        assert d.match(empty) == (a.q0, bool(a.accepting[a.q0]))
        x = torch.from_numpy(np.array([0, 1, 2, 3] * 100, np.uint8)).to(DEV)
        with pytest.raises(D.DfaError) as e:  # n < c + P - 1
            d.chunk_maps(x, 401)
        assert e.value.status == D.DFA_ERR_CHUNKS
        bad = np.array([0, 1, 2] * 1000 + [7] + [1] * 5000, np.uint8)  # byte 7 >= |Sigma| = 4
        with pytest.raises(D.DfaError) as e:
            d.match(torch.from_numpy(bad).to(DEV))
        assert e.value.status == D.DFA_ERR_SYMBOL
        d.chunk_maps(torch.from_numpy(bad).to(DEV), 100)
        torch.cuda.synchronize()
        assert D.dfa_get_last_device_error(d.h) == D.DFA_ERR_SYMBOL
        # handle still usable afterwards
        good = np.array([0, 1, 2, 0] * 50, np.uint8)
        assert d.match(torch.from_numpy(good).to(DEV))[0] == oracle.Dfa(a.table, a.q0, a.accepting).run(good)
    finally:
        d.close()


def test_error_state_paper_example(golden_dir):
    """Fig.ExampleDFA: the run enters q_E inside C_0; maps are all q_E (reading R1)."""
    import json, os
    g = json.load(open(os.path.join(golden_dir, "fig_example_dfa.json")))
    table = np.full((5, 2), 4, np.uint16)
    for s, lab, t in g["triples"]:
        table[s, g["symbols"][lab]] = t
    a = automata.Automaton(table, 0, np.arange(5) == 3)
    x = np.array([g["symbols"][ch] for ch in g["input"]], np.uint8)
    c = Case(a, x)
    info = check_chunk_maps(c, 3, 2, 1)  # c = I_max = 2: Fig.InputString
    assert info["i_max"] == 2
    big = np.tile(x, 5000)
    check_chunk_maps(Case(a, big), 999)


def test_match_host_equals_match():
    w = W.get("random")
    x = w.input(1 << 22)
    d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
    try:
        pinned = torch.from_numpy(x).pin_memory()
        assert D.dfa_match_host(d.h, pinned) == d.match(pinned.to(DEV))
        assert D.dfa_match_host(d.h, x) == d.match(pinned.to(DEV))
    finally:
        d.close()


def test_streams_and_repeat_determinism():
    w = W.get("protein")
    x = w.input(1 << 21)
    c = Case(w.automaton, x)
    d = c.handle()
    try:
        s = torch.cuda.Stream()
        dx = torch.from_numpy(x).to(DEV)
        with torch.cuda.stream(s):
            r1 = d.match(dx, stream=s)
        r2 = d.match(dx)
        assert r1 == r2 == (c.od.run(x), bool(c.a.accepting[c.od.run(x)]))
    finally:
        d.close()


# ------------------------------------------------------------------ full sizes (sampled)
def full_size(name, rows=4, seed=0):
    w = W.get(name, seed)
    x = w.input()
    c = Case(w.automaton, x, name)
    dx = torch.from_numpy(x).to(DEV)
    rng = np.random.default_rng(1)
    P = w.chunks
    rows_ = sorted(set([1, P - 1] + rng.integers(1, P, rows).tolist()))
    check_chunk_maps(c, P, dev=dx, maps_rows=rows_)
    d = c.handle()
    try:
        fin, acc = d.match(dx)
        assert fin == c.od.run(x)
    finally:
        d.close()


def test_full_random():
    full_size("random")


def test_full_keyword():
    full_size("keyword")


@pytest.mark.slow
def test_full_protein():
    full_size("protein", rows=2)


@pytest.mark.slow
def test_full_worst():
    full_size("worst", rows=2)


@pytest.mark.parametrize("fanin", [2, 3, 17, 64])
def test_tree_fanin(fanin):
    """The composition tree's shape must not change any result."""
    for name, n, P in (("random", 1 << 20, 1000), ("protein", 1 << 19, 300), ("tiny", 1 << 18, 64)):
        w = W.get(name)
        c = Case(w.automaton, w.input(n), name)
        check_chunk_maps(c, P, opts={D.DFA_OPT_TREE_FANIN: fanin, D.DFA_OPT_SUBCHUNK_TARGET: 5000})


@pytest.mark.parametrize("name,G", [("random", 4), ("keyword", 3), ("protein", 2), ("worst", 2), ("tiny", 8)])
def test_segment_maps_fold(name, G):
    """Sharded path kernels on one GPU: G segment maps (dfa_segment_map) folded
    by dfa_fold_segments == the sequential run; rows == the oracle's chunk maps."""
    w = W.get(name)
    check_segment_fold(Case(w.automaton, w.input(1 << 19), name), G)


@pytest.mark.parametrize("seed", range(4))
def test_segment_fold_small_alphabet_sink(seed):
    """|Sigma| < 256 with a user error state q_E: q_E is not internally absorbing (bytes
    >= |Sigma| lead to the poison state) but the fold must pass it through
    like any error state; the running state reaches q_E early (sink_frac 0.3)."""
    a = automata.random_dfa_with_sink(40, 20, seed, 0.3)
    rng = np.random.default_rng(seed)
    c = Case(a, rng.integers(0, 20, 1 << 19).astype(np.uint8), "sink")
    assert c.od.run(c.x) == 39  # the run ends in q_E
    check_segment_fold(c, 2 + seed)
    # the pipelined host path folds its pieces the same way
    d = c.handle({D.DFA_OPT_HOST_PIECE: 1 << 20})
    try:
        x3 = np.tile(c.x, 5)
        fin, acc = D.dfa_match_host(d.h, torch.from_numpy(x3).pin_memory())
        assert (fin, acc) == (c.od.run(x3), False)
    finally:
        d.close()


def check_segment_fold(c: Case, G: int):
    x = c.x
    n = x.size
    rng = np.random.default_rng(G)
    cuts = np.sort(rng.choice(np.arange(1, n), G - 1, replace=False))
    b = np.concatenate([[0], cuts, [n]]).astype(np.uint64)
    d = c.handle()
    try:
        imax = d.info["i_max"]
        dx = torch.from_numpy(x).to(DEV)
        rows = torch.empty(G, imax, dtype=torch.int16, device=DEV)
        la = np.zeros(G, np.uint8)
        for g in range(G):
            lo, hi = int(b[g]), int(b[g + 1])
            look = -1 if g == 0 else int(x[lo - 1])
            la[g] = max(look, 0)
            D.dfa_segment_map(d.h, dx[lo:hi], look, rows[g])
        final = torch.empty(2, dtype=torch.int16, device=DEV)
        D.dfa_fold_segments(d.h, rows, torch.from_numpy(la).to(DEV), G, final)
        torch.cuda.synchronize()
        assert D.dfa_get_last_device_error(d.h) == 0
        r = u16(rows)
        fin = c.od.run(x)
        assert u16(final).tolist() == [fin, int(c.a.accepting[fin])]
        assert r[0][0] == c.od.run(x[:int(b[1])])
        for g in range(1, G):
            row, _ = c.od.chunk_map(x, int(b[g]), int(b[g + 1]), imax)
            assert np.array_equal(r[g], row), g
    finally:
        d.close()


@pytest.mark.parametrize("off", [1, 5, 15, 31])
def test_misaligned_input(off):
    """Input pointers need no alignment (head bytes before the first 32-byte sector)."""
    for name in ("random", "protein"):
        w = W.get(name)
        x = w.input((1 << 18) + 77)
        full = torch.from_numpy(x).to(DEV)
        c = Case(w.automaton, x[off:], name)
        check_chunk_maps(c, 97, dev=full[off:])
        d = c.handle()
        try:
            assert d.match(full[off:])[0] == c.od.run(x[off:])
        finally:
            d.close()


def test_repeated_calls_graph_replay():
    """Identical repeated dfa_chunk_maps calls are replayed from a captured CUDA
    graph: results must stay identical to the oracle, also after changing buffers."""
    w = W.get("keyword")
    x = w.input(1 << 20)
    c = Case(w.automaton, x, "keyword")
    d = c.handle()
    try:
        dx = torch.from_numpy(x).to(DEV)
        ob = oracle.chunk_bounds_ratio(x.size, 300, 1, 1)
        oe0, omaps = c.od.maps(x, ob, d.info["i_max"])
        ofin = c.od.run(x)
        for rep in range(5):
            if rep == 3:  # new input buffer: new graph
                dx = dx.clone()
            bounds, e0, maps, starts, final = d.chunk_maps(dx, 300)
            torch.cuda.synchronize()
            assert u16(e0)[0] == oe0 and np.array_equal(u16(maps), omaps) and u16(final)[0] == ofin, rep
    finally:
        d.close()


# ------------------------------------------------------------------ N1: r-symbol reverse lookahead
def check_lookahead(c: Case, P: int, rs=(1, 2, 3, 4), bounds_in=None):
    """dfa_lookahead_maps against oracle.chunk_map_r, every chunk, every entry."""
    d = c.handle()
    try:
        x = c.x
        dx = torch.from_numpy(x).to(DEV)
        imax = d.info["i_max"]
        if bounds_in is None:
            bounds, e0, maps, _, _ = d.chunk_maps(dx, P)
        else:
            bounds = torch.from_numpy(np.asarray(bounds_in, np.int64)).to(DEV)
            e0 = torch.empty(1, dtype=torch.int16, device=DEV)
            maps = torch.empty(max(P - 1, 1) * imax, dtype=torch.int16, device=DEV)
            D.dfa_chunk_maps_at(d.h, dx, P, bounds, e0, maps)
            maps = maps.view(max(P - 1, 1), imax)[:P - 1]
        ob = bounds.cpu().numpy().astype(np.int64)
        for r in rs:
            doms, sizes, maps_r = d.lookahead_maps(dx, bounds, maps, r)
            torch.cuda.synchronize()
            assert D.dfa_get_last_device_error(d.h) == 0
            gd, gs, gm = u16(doms), u16(sizes), u16(maps_r)
            for k in range(1, P):
                dom, row, cnt = c.od.chunk_map_r(x, int(ob[k]), int(ob[k + 1]), r, imax)
                assert gs[k - 1] == cnt, f"r={r} chunk {k}: |domain| {gs[k - 1]} != {cnt}"
                assert np.array_equal(gd[k - 1], dom), f"r={r} chunk {k}: domain"
                assert np.array_equal(gm[k - 1], row), f"r={r} chunk {k}: map"
    finally:
        d.close()


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_lookahead_maps_configs(name):
    w = W.get(name)
    x = w.input(1 << 16)
    check_lookahead(Case(w.automaton, x, name), 97)


def test_lookahead_maps_short_prefix():
    """Chunks starting before offset r use the L = b_k < r available symbols."""
    w = W.get("keyword")
    x = w.input(4096)
    b = [0, 1, 2, 3, 5, 8, 13, 100, 1000, 4096]
    check_lookahead(Case(w.automaton, x, "keyword"), len(b) - 1, rs=(1, 2, 4, 16), bounds_in=b)


def test_lookahead_maps_sink_and_small_alphabet():
    for seed in range(3):
        a = automata.random_dfa_with_sink(40, 5, seed)
        x = np.random.default_rng(seed).integers(0, 5, 3000).astype(np.uint8)
        check_lookahead(Case(a, x, f"sink{seed}"), 31, rs=(1, 2, 3, 5))


# ------------------------------------------------------------------ N2: Alg. 2 ablation (all of Q minus Z)
@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_alg2_full_domain_parity(name):
    """DFA_CREATE_FULL_DOMAIN matches every sub-chunk from Q minus Z (Alg.2):
    identical results, including the API rows over I_sigma."""
    w = W.get(name)
    x = w.input(min(w.small_n, 1 << 20))
    c = Case(w.automaton, x, name)
    check_chunk_maps(c, 61, flags=D.DFA_CREATE_FULL_DOMAIN)
    check_match(c, flags=D.DFA_CREATE_FULL_DOMAIN)


# ------------------------------------------------------------------ sticky-lane parking (lanes_kernel)
def sticky_dfa(nq: int, seed: int, n_kill: int = 6, die_rate: float = 0.05):
    """Random DFA over 256 bytes with a dead sink (state nq-1), universal kill bytes
    (the last n_kill byte values send every state to the sink), a sticky state 0
    (every other byte keeps it) and random states that also die on some ordinary bytes."""
    rng = np.random.default_rng(seed)
    sink = nq - 1
    t = rng.integers(1, nq - 1, size=(nq, 256)).astype(np.uint16)
    t[rng.random((nq, 256)) < die_rate] = sink
    t[0, :] = 0
    t[:, 256 - n_kill:] = sink
    t[sink, :] = sink
    # make state 0 reachable from many states on a few bytes
    t[:, 10] = np.where(np.arange(nq) == sink, sink, 0)
    acc = [0, 3]
    return automata.Automaton(t, 0 if seed % 2 else 1, np.array([q in acc for q in range(nq)]),
                              f"sticky{seed}")


@pytest.mark.parametrize("seed", range(6))
def test_sticky_parking(seed):
    """Parked lanes survive while a witness lives, die with it on a kill byte, and
    resume from the parking offset when the witness ends on an ordinary byte."""
    a = sticky_dfa(12 + 5 * seed, seed)
    rng = np.random.default_rng(100 + seed)
    n = 1 << 18
    x = rng.integers(0, 250, n).astype(np.uint8)
    # sparse kill bytes and dense runs of the byte that enters the sticky state
    kills = rng.choice(n, 8 + seed * 4, replace=False)
    x[kills] = rng.integers(250, 256, kills.size)
    x[rng.choice(n, 2000, replace=False)] = 10
    c = Case(a, x, f"sticky{seed}")
    for P in (1, 7, 333):
        check_chunk_maps(c, P)
    check_match(c)


@pytest.mark.parametrize("cap", [1, 3, 5])
@pytest.mark.parametrize("name", ["random", "keyword", "protein", "worst"])
def test_max_lanes(name, cap):
    """DFA_OPT_MAX_LANES (the Worst config's lanes-per-thread sweep): converge to
    <= cap survivors / several passes of <= cap lanes; same results."""
    w = W.get(name)
    x = w.input(min(w.small_n, 1 << 19))
    c = Case(w.automaton, x, name)
    check_chunk_maps(c, 129, opts={D.DFA_OPT_MAX_LANES: cap})


# ------------------------------------------------------------------ shared-memory table layouts
@pytest.mark.parametrize("mode", [1, 7, 8, 9])
def test_table_layouts(mode):
    """IdentU8, its bank-group replicas (R = 8, 4 copies) and its padded-row form
     give identical results: the five-config DFAs that fit, a small-alphabet DFA
    with a sink (poison state), a sticky-parking DFA and misaligned input."""
    flags = D.DFA_CREATE_TABLE_MODE(mode)
    cases = []
    for name in ("tiny", "random", "keyword"):
        w = W.get(name)
        cases.append((Case(w.automaton, w.input(min(w.small_n, 1 << 19)), name), 129))
    rng = np.random.default_rng(7)
    a = automata.random_dfa_with_sink(40, 20, 7, 0.3)
    cases.append((Case(a, rng.integers(0, 20, 300001).astype(np.uint8), "sink"), 77))
    s = sticky_dfa(30, 3)
    xs = rng.integers(0, 250, 1 << 18).astype(np.uint8)
    xs[rng.choice(xs.size, 2000, replace=False)] = 10
    xs[rng.choice(xs.size, 9, replace=False)] = 255
    cases.append((Case(s, xs, "sticky"), 333))
    for c, P in cases:
        info = check_chunk_maps(c, P, flags=flags)
        nq = c.a.table.shape[0] + (1 if c.a.table.shape[1] < 256 else 0)
        want = {1: "ident_u8", 7: "rep8_u8" if nq * 2048 + 2048 <= 223 * 1024 else "ident_u8_pad",
                8: "rep4_u8" if nq * 1024 + 1024 <= 223 * 1024 else "ident_u8_pad", 9: "ident_u8_pad"}[mode]
        assert info["table_mode_name"] == want, (c.name, info["table_mode_name"])
        check_match(c, flags=flags)
    # misaligned device input
    w = W.get("random")
    x = w.input(1 << 20)
    buf = torch.from_numpy(np.concatenate([np.zeros(5, np.uint8), x])).to(DEV)
    check_chunk_maps(Case(w.automaton, x, "random+5"), 300, dev=buf[5:], flags=flags)


def test_window_fast_and_slow_paths():
    """WindowU16 (|Q| > 252, the non-default bytes inside one aligned window): 16-byte
    blocks entirely inside the window take the low-bits column step, blocks with an
    outside byte the clamped one; mixed per warp, same results."""
    rng = np.random.default_rng(11)
    nq = 300
    t = rng.integers(0, nq, size=(nq, 256)).astype(np.uint16)
    t[:, :64] = t[:, [200]]          # every byte outside [64, 128) behaves like byte 200
    t[:, 128:] = t[:, [200]]
    a = automata.Automaton(t, 0, rng.random(nq) < 0.3, "window")
    n = 1 << 19
    x = rng.integers(64, 128, n).astype(np.uint8)
    out = rng.random(n) < 0.02
    x[out] = rng.integers(0, 256, int(out.sum()))
    c = Case(a, x, "window")
    for P in (1, 97, 1000):
        info = check_chunk_maps(c, P)
        assert info["table_mode_name"] == "window_u16", info["table_mode_name"]
    check_match(c)


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_gather_ceiling_kernel(name):
    """dfa_gather_ceiling (measurement aid): thread t's output is delta-hat(q0, its bytes)."""
    w = W.get(name)
    x = w.input(min(w.small_n, 1 << 22))
    dx = torch.from_numpy(x).to(DEV)
    d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
    try:
        nt, per = D.dfa_gather_ceiling(d.h, dx, None)
        if per == 0:
            x = np.tile(x, 32 * nt // x.size + 1)[:32 * nt * 2]
            dx = torch.from_numpy(x).to(DEV)
            nt, per = D.dfa_gather_ceiling(d.h, dx, None)
        assert per > 0 and per % 32 == 0
        out = torch.empty(nt, dtype=torch.int16, device=DEV)
        D.dfa_gather_ceiling(d.h, dx, out)
        torch.cuda.synchronize()
        got = u16(out)
        od = oracle.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accepting)
        for t in (0, 1, nt // 2, nt - 1):
            assert got[t] == od.run(x[t * per:(t + 1) * per]), t
        with pytest.raises(D.DfaError):
            D.dfa_gather_ceiling(d.h, dx[1:], out, length=x.size - 1)  # misaligned
    finally:
        d.close()


# ------------------------------------------------------------------ dfa_match_host pipeline + early exit (N4)
@pytest.mark.parametrize("name", ["random", "keyword", "protein", "tiny"])
@pytest.mark.parametrize("early", [0, 1])
def test_match_host_pipelined(name, early):
    """Pieces of 1 MiB (the last ragged): same final/accept as the oracle; with early
    exit the bytes copied stop once the running state absorbs every byte."""
    w = W.get(name)
    x = w.input((5 << 20) + 12345)
    c = Case(w.automaton, x, name)
    d = c.handle({D.DFA_OPT_HOST_PIECE: 1 << 20, D.DFA_OPT_EARLY_EXIT: early})
    try:
        pinned = torch.from_numpy(x).pin_memory()
        fin, acc = D.dfa_match_host(d.h, pinned)
        ofin = c.od.run(x)
        assert (fin, acc) == (ofin, bool(c.a.accepting[ofin]))
        copied = D.dfa_get_stats(d.h)["host_bytes"]
        assert copied <= x.size
        if not early:
            assert copied == x.size
    finally:
        d.close()


def test_match_host_early_exit_stops():
    """Keyword DFA (absorbing accept): a keyword in the first piece ends the copy early;
    a bad-free input without keywords is copied whole."""
    w = W.get("keyword")
    a = w.automaton
    kw = np.frombuffer(w.info["keywords"][0].encode("latin1"), np.uint8)
    x = np.full((8 << 20) + 7, 0x20, np.uint8)  # spaces: no keyword
    c = Case(a, x, "kw-none")
    d = c.handle({D.DFA_OPT_HOST_PIECE: 1 << 20})
    try:
        fin, acc = D.dfa_match_host(d.h, x)
        assert (fin, acc) == (c.od.run(x), bool(a.accepting[c.od.run(x)]))
        assert D.dfa_get_stats(d.h)["host_bytes"] == x.size
        y = x.copy()
        y[1000:1000 + kw.size] = kw
        fin, acc = D.dfa_match_host(d.h, y)
        assert acc and fin == c.od.run(y)
        assert D.dfa_get_stats(d.h)["host_bytes"] < y.size
    finally:
        d.close()


# ------------------------------------------------------------------ dfa_match_batch (N4 multi-input batching)
def check_batch(c: Case, lengths, seed=0):
    rng = np.random.default_rng(seed)
    ns = c.a.table.shape[1]
    offs = np.concatenate([[0], np.cumsum(lengths)]).astype(np.uint64)
    data = rng.integers(0, ns, int(offs[-1]) + 1).astype(np.uint8)
    d = c.handle()
    try:
        dd = torch.from_numpy(data).to(DEV)
        fin = torch.empty(len(lengths), dtype=torch.int16, device=DEV)
        acc = torch.empty(len(lengths), dtype=torch.uint8, device=DEV)
        D.dfa_match_batch(d.h, dd, torch.from_numpy(offs.astype(np.int64)).to(DEV), fin, acc)
        torch.cuda.synchronize()
        assert D.dfa_get_last_device_error(d.h) == 0
        gf, ga = u16(fin), acc.cpu().numpy()
        idx = range(len(lengths))
        if len(lengths) > 20000:  # every input's result is independent: a seeded sample + both ends
            idx = sorted(set(rng.choice(len(lengths), 20000, replace=False).tolist()) | {0, len(lengths) - 1})
        for j in idx:
            x = data[int(offs[j]):int(offs[j + 1])]
            of = c.od.run(x)
            assert gf[j] == of and ga[j] == int(c.a.accepting[of]), f"input {j} (len {x.size})"
    finally:
        d.close()


@pytest.mark.parametrize("nq,ns", [(40, 256), (80, 256), (109, 20)])
def test_rep8_with_converge_stage(nq, ns):
    """rep8_u8 (640-thread lanes kernel) on DFAs whose I_max > 8, so the converge kernel
    (padded single copy) hands survivors to the replicated-table lanes kernel: chunk maps,
    host-input pipeline and batches against the oracle."""
    a = automata.random_dfa(nq, ns, 1000 + nq)
    rng = np.random.default_rng(nq)
    x = rng.integers(0, ns, 700001).astype(np.uint8)
    c = Case(a, x, f"rep8conv{nq}")
    d = c.handle()
    try:
        assert d.info["table_mode_name"] == "rep8_u8" and d.info["i_max"] > 8, d.info
        D.dfa_set_option(d.h, D.DFA_OPT_HOST_PIECE, 1 << 20)  # several pipelined pieces
        fin, acc = D.dfa_match_host(d.h, x)
        assert fin == c.od.run(x)
    finally:
        d.close()
    for P in (1, 33, 4000):
        check_chunk_maps(c, P)
    check_batch(c, [0, 1, 31, 32, 33, 1000, 4097] * 50, seed=nq)


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_match_batch_many_small(name):
    w = W.get(name)
    rng = np.random.default_rng(5)
    lengths = rng.integers(0, 700, 5000)
    lengths[rng.random(5000) < 0.05] = 0
    check_batch(Case(w.automaton, np.zeros(1, np.uint8), name), lengths)


@pytest.mark.parametrize("name", ["random", "protein", "worst"])
def test_match_batch_few_large(name):
    w = W.get(name)
    check_batch(Case(w.automaton, np.zeros(1, np.uint8), name), [300000, 0, 1, 123457, 65536], seed=2)


def test_match_batch_bad_offsets():
    w = W.get("random")
    d = Case(w.automaton, np.zeros(1, np.uint8), "random").handle()
    try:
        dd = torch.zeros(1000, dtype=torch.uint8, device=DEV)
        fin = torch.empty(5000, dtype=torch.int16, device=DEV)
        acc = torch.empty(5000, dtype=torch.uint8, device=DEV)
        off = torch.arange(5001, dtype=torch.int64, device=DEV) % 1200  # decreasing and past the data
        D.dfa_match_batch(d.h, dd, off, fin, acc)
        torch.cuda.synchronize()
        assert D.dfa_get_last_device_error(d.h) == D.DFA_ERR_ARG
        bad = torch.tensor([0, 10, 5, 20], dtype=torch.int64, device=DEV)
        with pytest.raises(D.DfaError):
            D.dfa_match_batch(d.h, dd, bad, fin, acc)  # few inputs: validated on the host
        past = torch.tensor([0, 10, 2000], dtype=torch.int64, device=DEV)
        with pytest.raises(D.DfaError):
            D.dfa_match_batch(d.h, dd, past, fin, acc)
    finally:
        d.close()


def _nccl_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    from paper_1210_5093_b200 import multi_gpu
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        res = []
        for name in ("random", "protein", "keyword"):
            w = W.get(name)
            x = w.input(1 << 20, segment=rank)
            dx = torch.from_numpy(x).cuda()
            d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
            smap, fold = multi_gpu.gpu_ops(d, dx)
            m = multi_gpu.SegmentMatcher(rank, world, dist, dx[-1:], smap, fold)
            row = m.step()  # world 1: the segment row (entry 0 = final state), no collective
            # the N > 1 exchange over NCCL anyway: all-gather of the rows, then the fold kernel
            out = fold(multi_gpu.gather_rows(row, dist), [-1])
            torch.cuda.synchronize()
            res.append((name, out.cpu().numpy().view(np.uint16).tolist(), D.dfa_get_last_device_error(d.h)))
            d.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharded_path_nccl_world1():
    """The N > 1 bench path (segment map -> NCCL all-gather -> fold) end to end over
    NCCL on this GPU with world size 1 (one process per GPU; the box has one)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(0, 1, port, q))
    p.start()
    rank, res = q.get(timeout=300)
    p.join(60)
    for name, fin, err in res:
        w = W.get(name)
        od = oracle.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accepting)
        f = od.run(w.input(1 << 20))
        assert err == 0 and fin == [f, int(w.automaton.accepting[f])], name


# ------------------------------------------------------------------ round-2 hygiene: graph replay, limits, options
def test_graph_replay_alternating_chunk_counts():
    """A captured graph must never replay stale scratch: alternate P values (which
    reallocate scratch and reshape the composition tree) with fixed output buffers."""
    for name in ("random", "protein"):
        w = W.get(name)
        x = w.input(1 << 20)
        c = Case(w.automaton, x, name)
        d = c.handle()
        try:
            dx = torch.from_numpy(x).to(DEV)
            imax = d.info["i_max"]
            outs = {}
            for P in (300, 65536):
                outs[P] = (torch.empty(P + 1, dtype=torch.int64, device=DEV),
                           torch.empty(1, dtype=torch.int16, device=DEV),
                           torch.empty((P - 1) * imax, dtype=torch.int16, device=DEV),
                           torch.empty(2, dtype=torch.int16, device=DEV))
            want = {}
            for P in outs:
                ob = oracle.chunk_bounds_ratio(x.size, P, 1, 1)
                want[P] = c.od.maps(x, ob, imax)
            fin = c.od.run(x)
            for P in (300, 300, 300, 65536, 300, 65536, 65536, 65536, 300, 300):
                b, e0, maps, final = outs[P]
                maps.fill_(0)
                D.dfa_chunk_maps(d.h, dx, P, b, e0, maps, None, final)
                torch.cuda.synchronize()
                assert D.dfa_get_last_device_error(d.h) == 0
                oe0, omaps = want[P]
                assert u16(e0)[0] == oe0 and u16(final)[0] == fin, (name, P)
                assert np.array_equal(u16(maps).reshape(omaps.shape), omaps), (name, P)
        finally:
            d.close()


def test_more_than_2_20_chunks():
    """P > 2^20 reporting chunks (compose8's limit) take the tree path; a batch of more
    than 2^20 inputs likewise."""
    w = W.get("random")
    x = w.input(3 << 20)
    c = Case(w.automaton, x, "random")
    check_chunk_maps(c, (1 << 20) + 3)
    check_batch(c, [2] * ((1 << 20) + 5), seed=3)


def test_sticky_parking_option_off():
    """DFA_OPT_STICKY_PARKING = 0 (the plain lanes kernel on a DFA with sticky states)."""
    w = W.get("protein")
    c = Case(w.automaton, w.input(1 << 20), "protein")
    check_chunk_maps(c, 300, opts={D.DFA_OPT_STICKY_PARKING: 0})
    check_chunk_maps(c, 300, opts={D.DFA_OPT_STICKY_PARKING: 1})


@pytest.mark.parametrize("name", ["tiny", "random", "keyword"])
def test_work_counter_is_L_alg(name):
    """DFA_OPT_COUNT_WORK with convergence off and one execution sub-chunk per chunk
    (dfa_chunk_maps_at): the lanes kernel's executed lane-steps are exactly L_alg =
    len_0 + sum_k len_k |I_sigma_k| (Alg.3 runs |I_sigma| lanes over its
    chunk; an empty I_sigma still steps one lane)."""
    w = W.get(name)
    x = w.input(1 << 20)
    c = Case(w.automaton, x, name)
    d = c.handle({D.DFA_OPT_CONVERGENCE: 0, D.DFA_OPT_COUNT_WORK: 1})
    try:
        P = 777
        ob = oracle.chunk_bounds_ratio(x.size, P, 1, 1).astype(np.int64)
        bounds = torch.from_numpy(ob).to(DEV)
        imax = d.info["i_max"]
        e0 = torch.empty(1, dtype=torch.int16, device=DEV)
        maps = torch.empty((P - 1) * imax, dtype=torch.int16, device=DEV)
        D.dfa_get_stats(d.h)
        D.dfa_chunk_maps_at(d.h, torch.from_numpy(x).to(DEV), P, bounds, e0, maps)
        torch.cuda.synchronize()
        st = D.dfa_get_stats(d.h)
        sizes = np.array([len(c.od.initial_states(int(s))) if s < w.automaton.ns else 0 for s in range(256)], np.int64)
        lens = np.diff(ob)
        L = int(lens[0] + (lens[1:] * np.maximum(sizes[x[ob[1:-1] - 1]], 1)).sum())
        assert st["work"]["lanes"] == L and st["work"]["converge"] == 0 and st["work"]["calls"] == 1
        # convergence on: executed work is below L_alg and at least n
        D.dfa_set_option(d.h, D.DFA_OPT_CONVERGENCE, 1)
        D.dfa_chunk_maps_at(d.h, torch.from_numpy(x).to(DEV), P, bounds, e0, maps)
        torch.cuda.synchronize()
        st = D.dfa_get_stats(d.h)
        assert x.size <= st["work"]["lanes"] <= L
    finally:
        d.close()


@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("name", ["tiny", "random", "keyword"])
def test_fused_tail_and_compose8(name, fused):
    """Maps of <= 8 entries: the match kernel's fused composition tail (default) and the
    separate leaf_fold + compose8 launches (DFA_OPT_FUSED_TAIL = 0) give the oracle's
    bounds, e0, every map entry, every chunk start and the final state -- one chunk
    spanning every CTA (P = 1, 2), chunks straddling CTA boundaries, many chunks per CTA."""
    w = W.get(name)
    x = w.input(min(w.small_n, 1 << 21) + 4321)
    c = Case(w.automaton, x, name)
    for P in (1, 2, 3, 64, 777, 4096):
        check_chunk_maps(c, P, opts={D.DFA_OPT_FUSED_TAIL: fused})
    check_match(c, opts={D.DFA_OPT_FUSED_TAIL: fused})


def test_tma_input_staging():
    """DFA_OPT_TMA_INPUT = 1 (rep8_u8: the match kernel's input staged by TMA gather4 copies,
    run_lanes_tma): the oracle's maps, starts and final for chunk counts that leave whole and
    partial warps, sub-chunks shorter than a stage, a misaligned input pointer (rows from the
    32-byte aligned base) and an input whose last block's row would end past it."""
    w = W.get("random")
    for n in (1 << 20, (1 << 20) + 4321, 5000, 97):
        x = w.input(n)
        c = Case(w.automaton, x, "random")
        for P in (1, 3, 64, 777):
            if P <= n:
                info = check_chunk_maps(c, P, opts={D.DFA_OPT_TMA_INPUT: 1})
                assert info["table_mode_name"] == "rep8_u8"
        check_match(c, opts={D.DFA_OPT_TMA_INPUT: 1})
    x = w.input((1 << 19) + 77)
    c = Case(w.automaton, x, "random")
    buf = torch.zeros(x.size + 64, dtype=torch.uint8, device=DEV)
    for off in (1, 13, 32, 47):
        dev = buf[off:off + x.size]
        dev.copy_(torch.from_numpy(x))
        check_chunk_maps(c, 300, opts={D.DFA_OPT_TMA_INPUT: 1}, dev=dev)


@pytest.mark.parametrize("factored", [0, 1])
@pytest.mark.parametrize("name", ["worst", "protein", "counter"])
def test_factored_and_full_row_composition(name, factored):
    """Maps of more than 16 entries behind the converge stage: the factored composition
    (DFA_OPT_FACTORED = 1, the first sub-chunk's converge map then <= 8 survivor values per
    node) and the full-row walk give the oracle's maps, starts and final -- long sub-chunks
    (every node factored), chunks shorter than the convergence length (sub-chunks that end
    inside converge_kernel: FULL nodes, also as a node's first child), a DFA whose lanes never
    merge, several tree shapes (fan-in, sub-chunk targets)."""
    if name == "counter":
        a, x = automata.counter_dfa(37), inputs.uniform_bytes((1 << 19) + 77, seed=9)
    else:
        w = W.get(name)
        a, x = w.automaton, w.input((1 << 20) + 1234)
    c = Case(a, x, name)
    for P, extra in ((1, {}), (2, {}), (17, {}), (300, {D.DFA_OPT_TREE_FANIN: 3}), (4099, {}),
                     (33, {D.DFA_OPT_SUBCHUNK_TARGET: 5000}), (x.size // 24, {}),
                     (x.size // 150, {D.DFA_OPT_SUBCHUNK_TARGET: 1 << 22, D.DFA_OPT_TREE_FANIN: 5})):
        check_chunk_maps(c, P, opts={D.DFA_OPT_FACTORED: factored, **extra})
        if factored:  # internal sub-chunks from I_sigma instead of the two-symbol sets (Eq.istatesm)
            check_chunk_maps(c, P, opts={D.DFA_OPT_LOOKAHEAD2: 0, **extra})
    check_match(c, opts={D.DFA_OPT_FACTORED: factored})


@pytest.mark.parametrize("name,G,P", [("random", 3, 64), ("keyword", 2, 129), ("protein", 2, 33), ("worst", 2, 17),
                                      ("tiny", 4, 16)])
def test_segment_chunk_maps(name, G, P):
    """dfa_segment_chunk_maps (the per-GPU step of every N, Fig.Merge): for each
    of G segments of one input, P chunks with chunk 0 from I_sigma of the byte before the
    segment (segment 0 from q0): bounds, chunk 0's row (e0 for segment 0), every map row and
    the segment's composed row against the oracle; the rows fold to the sequential final."""
    w = W.get(name)
    n = 3 << 19
    x = w.input(n)
    c = Case(w.automaton, x, name)
    rng = np.random.default_rng(G + P)
    cuts = np.sort(rng.choice(np.arange(P + 1, n - P - 1), G - 1, replace=False))
    b = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    d = c.handle()
    try:
        imax = d.info["i_max"]
        dx = torch.from_numpy(x).to(DEV)
        rows = torch.empty(G, imax, dtype=torch.int16, device=DEV)
        la = np.zeros(G, np.uint8)
        for rep in range(2):  # the second pass replays captured graphs
            for g in range(G):
                lo, hi = int(b[g]), int(b[g + 1])
                look = -1 if g == 0 else int(x[lo - 1])
                la[g] = max(look, 0)
                bounds = torch.empty(P + 1, dtype=torch.int64, device=DEV)
                c0 = torch.empty(imax, dtype=torch.int16, device=DEV)
                maps = torch.empty((P - 1) * imax, dtype=torch.int16, device=DEV)
                D.dfa_segment_chunk_maps(d.h, dx[lo:hi], P, look, bounds, c0, maps, rows[g])
                torch.cuda.synchronize()
                assert D.dfa_get_last_device_error(d.h) == 0
                ob = oracle.chunk_bounds_ratio(hi - lo, P, 1, 1)
                assert np.array_equal(bounds.cpu().numpy().astype(np.uint64), ob), (g, "bounds")
                xs = x[lo:hi]
                oe0, omaps = c.od.maps(xs, ob, imax)
                assert np.array_equal(u16(maps).reshape(omaps.shape), omaps), (g, "maps")
                if g == 0:
                    assert u16(c0)[0] == oe0, "e0"
                    assert u16(rows[0])[0] == c.od.run(xs), "segment 0 final"
                else:
                    row0, _ = c.od.chunk_map(x, lo, lo + int(ob[1]), imax)
                    assert np.array_equal(u16(c0), row0), (g, "chunk 0 row")
                    srow, _ = c.od.chunk_map(x, lo, hi, imax)
                    assert np.array_equal(u16(rows[g]), srow), (g, "segment row")
        final = torch.empty(2, dtype=torch.int16, device=DEV)
        D.dfa_fold_segments(d.h, rows, torch.from_numpy(la).to(DEV), G, final)
        torch.cuda.synchronize()
        fin = c.od.run(x)
        assert u16(final).tolist() == [fin, int(c.a.accepting[fin])]
    finally:
        d.close()

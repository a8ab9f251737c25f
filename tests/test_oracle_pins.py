"""Pins for the CPU oracle: values the paper prints, closed forms, brute force
and invariants -- never the oracle's own formula retyped.  (-m "not gpu")."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from oracle import Dfa
from workloads import automata, inputs


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def motiv_dfa(g, q0=None):
    return Dfa(g["table"], g["q0"] if q0 is None else q0, g["final_states"])


def enc(text, symbols):
    return np.array([symbols[ch] for ch in text], np.uint8)


def example_dfa(g):
    table = np.full((5, 2), g["missing_transitions_go_to"], np.uint16)
    for s, lab, d in g["triples"]:
        table[s, g["symbols"][lab]] = d
    return Dfa(table, g["q0"], g["final_states"])


# --------------------------------------------------------------------------- P1
def test_motiv_dfa_final_and_accept(golden_dir):
    g = load(golden_dir, "fig_motiv_dfa.json")
    d = motiv_dfa(g)
    x = enc(g["input"], g["symbols"])
    assert d.run(x) == g["expected_final"]
    assert d.accepts(x) is g["expected_accept"]


def test_motiv_dfa_equal_chunk_maps(golden_dir):
    """Fig.naive: chunks matched from every non-error state; L2 = [qE, q1]."""
    g = load(golden_dir, "fig_motiv_dfa.json")
    x = enc(g["input"], g["symbols"])
    (b1, e1), (b2, e2) = g["equal_chunks"][1], g["equal_chunks"][2]
    L1 = [motiv_dfa(g, q).run(x[b1:e1]) for q in (0, 1)]
    L2 = [motiv_dfa(g, q).run(x[b2:e2]) for q in (0, 1)]
    assert L1 == g["L1_over_q0_q1"]
    assert L2 == g["L2_over_q0_q1"]
    # Eq.SeqReduction over the dense maps: L2[L1[L0[0]]]
    e0 = motiv_dfa(g).run(x[:4])
    assert L2[L1[e0]] == g["expected_final"]


def test_motiv_dfa_initial_state_sets(golden_dir):
    g = load(golden_dir, "fig_motiv_dfa.json")
    d = motiv_dfa(g)
    for sym in "abc":
        assert d.initial_states(g["symbols"][sym]).tolist() == g["I_" + sym]
    assert d.dead.tolist() == [0, 0, 1]
    assert d.imax() == 1  # best case I_max = 1


# --------------------------------------------------------------------------- P2
def test_example_dfa_initial_sets_and_imax(golden_dir):
    g = load(golden_dir, "fig_example_dfa.json")
    d = example_dfa(g)
    assert d.initial_states(0).tolist() == g["I_a"]
    assert d.initial_states(1).tolist() == g["I_b"]
    assert d.imax() == g["I_max"]
    assert d.dead.tolist() == [0, 0, 0, 0, 1]


def _inclusive(b):
    return [[int(b[k]), int(b[k + 1]) - 1] for k in range(len(b) - 1)]


def test_example_dfa_bounds(golden_dir):
    """Fig.InputString (m = I_max = 2) and the unoptimised m = |Q| = 4."""
    g = load(golden_dir, "fig_example_dfa.json")
    b2 = oracle.chunk_bounds(g["n"], 3, 2)
    assert _inclusive(b2) == g["bounds_m2_inclusive"]
    assert int(b2[1]) == 18  # l0 = 18
    x = g["input"]
    assert [x[b2[k]:b2[k + 1]] for k in range(3)] == g["chunk_texts_m2"]
    assert [x[b2[k] - 1] for k in (1, 2)] == g["lookahead_symbols_m2"]
    b4 = oracle.chunk_bounds(g["n"], 3, 4)
    assert _inclusive(b4) == g["bounds_m4_inclusive"]
    assert int(b4[1]) == 24


def test_example_dfa_run_maps_fold(golden_dir):
    """The running example ends in the error state; every map is all-qE, the true
    start of C1 is qE (not in I_a) and the fold still recovers it (reading R1)."""
    g = load(golden_dir, "fig_example_dfa.json")
    d = example_dfa(g)
    x = enc(g["input"], g["symbols"])
    assert d.run(x) == 4
    b = oracle.chunk_bounds(g["n"], 3, 2)
    e0, maps = d.maps(x, b, 2)
    assert e0 == 4
    assert maps.tolist() == [[4, 4], [4, 4]]
    assert d.fold(x, b, 2, e0, maps) == 4
    starts, fin = d.run_record(x, b[:-1])
    assert starts.tolist() == [0, 4, 4] and fin == 4


# --------------------------------------------------------------------------- P3
def test_table_example_chunk_comp(golden_dir):
    g = load(golden_dir, "tab_example_chunk_comp.json")
    b = oracle.chunk_bounds(g["n"], 3, g["m"], g["capacities"])
    assert _inclusive(b) == g["ranges_inclusive"]
    # c-form: c = w0*m/w = 1.5*4/0.75 = 8 gives the same partition
    assert oracle.chunk_bounds_ratio(g["n"], 3, 8, 1).tolist() == b.tolist()


# --------------------------------------------------------------------------- P4
def test_sbase_ibase(golden_dir):
    g = load(golden_dir, "fig_sbase_example.json")
    e = load(golden_dir, "fig_example_dfa.json")
    d = example_dfa(e)
    assert d.table.ravel().tolist() == g["SBase"]
    x = enc(g["input"], e["symbols"])
    assert x.tolist() == g["IBase"]
    assert d.run(x) == g["derived_final"]


# --------------------------------------------------------------------------- P5
def _contains(s, kws):
    return any(kws_i in s for kws_i in kws)


def test_tiny_dfa_brute_force_all_short_strings():
    """accept <=> 'abca' or 'bdd' is a substring, for all 87,381 strings of length <= 8;
    if rejected, the final state is the longest suffix that is a proper keyword prefix."""
    aut = automata.aho_corasick([[0, 1, 2, 0], [1, 3, 3]], 4)
    d = Dfa(aut.table, aut.q0, aut.accepting)
    prefixes = {(): 0, (0,): 1, (1,): 2, (0, 1): 3, (1, 3): 4, (0, 1, 2): 5}
    kws = ["abca", "bdd"]
    count = 0
    for L in range(0, 9):
        for t in itertools.product(range(4), repeat=L):
            x = np.array(t, np.uint8)
            s = "".join("abcd"[i] for i in t)
            acc = _contains(s, kws)
            fin = d.run(x)
            assert bool(d.accepting[fin]) == acc, s
            if not acc:
                best = max((p for p in prefixes if len(p) <= L and tuple(t[L - len(p):]) == p),
                           key=len)
                assert fin == prefixes[best], s
            count += 1
    assert count == 87381


def test_keyword_dfa_vs_naive_search():
    kws = inputs.random_keywords(8, seed=3, lo=2, hi=4, first=0x61, last=0x64)
    aut = automata.aho_corasick([list(k) for k in kws], 256)
    d = Dfa(aut.table, aut.q0, aut.accepting)
    rng = np.random.default_rng(5)
    for _ in range(3000):
        L = int(rng.integers(0, 24))
        x = rng.integers(0x61, 0x65, L).astype(np.uint8)
        if rng.random() < 0.1 and L:
            x[int(rng.integers(L))] = int(rng.integers(0, 256))
        s = bytes(x.tolist())
        assert d.accepts(x) == any(k in s for k in kws)


def _motif_match_at(seq, motif, i, p=0):
    if p == len(motif):
        return True
    kind, allowed, lo, hi = motif[p]
    for L in range(lo, hi + 1):
        if i + L > len(seq):
            break
        if all(c in allowed for c in seq[i:i + L]) and _motif_match_at(seq, motif, i + L, p + 1):
            return True
    return False


def test_motif_dfa_vs_backtracking():
    rng = np.random.Generator(np.random.Philox(key=11))
    motif = [("res", {0}, 1, 1), ("gap", set(range(20)), 2, 4), ("class", {1, 2}, 1, 1),
             ("excl", set(range(20)) - {3}, 1, 1), ("res", {4}, 1, 1)]
    aut = automata.extend_to_bytes(automata.motif_dfa_residues(motif), automata.RESIDUES)
    d = Dfa(aut.table, aut.q0, aut.accepting)
    res = np.frombuffer(automata.RESIDUES, np.uint8)
    for _ in range(1500):
        L = int(rng.integers(0, 40))
        idx = rng.integers(0, 6, L)  # small sub-alphabet so matches happen
        seq = idx.tolist()
        x = res[idx]
        foreign = rng.random() < 0.05 and L > 0
        if foreign:
            x = x.copy()
            x[int(rng.integers(L))] = ord("B")
        expect = (not foreign) and any(_motif_match_at(seq, motif, i) for i in range(L + 1))
        assert d.accepts(x) == expect


def test_counter_dfa_closed_form():
    """delta(q,c) = (q+c) mod |Q|: final = (q0 + sum x) mod |Q|; chunk maps are shifts."""
    nq = 37
    aut = automata.counter_dfa(nq)
    d = Dfa(aut.table, 5, aut.accepting)
    x = inputs.uniform_bytes(100_000, seed=9)
    assert d.run(x) == (5 + int(x.astype(np.int64).sum())) % nq
    # every column is a permutation -> I_sigma = Q, gamma = 1
    assert d.imax() == nq
    b = oracle.chunk_bounds(x.size, 7, nq)
    e0, maps = d.maps(x, b, nq)
    assert e0 == (5 + int(x[:b[1]].astype(np.int64).sum())) % nq
    for k in range(1, 7):
        shift = int(x[b[k]:b[k + 1]].astype(np.int64).sum())
        assert maps[k - 1].tolist() == [(j + shift) % nq for j in range(nq)]


def test_reset_and_identity_closed_forms():
    rng = np.random.default_rng(1)
    f = rng.integers(0, 10, 256)
    d = Dfa(automata.reset_dfa(10, f).table, 0, [1])
    x = inputs.uniform_bytes(5000, seed=2)
    assert d.run(x) == f[x[-1]]
    for s in range(256):
        assert d.initial_states(s).tolist() == [f[s]]
    idd = Dfa(automata.identity_dfa(6).table, 4, [4])
    assert idd.run(x) == 4
    assert idd.run(x[:0]) == 4


# --------------------------------------------------------------------------- P6
def _random_partition(rng, n, P):
    cuts = np.sort(rng.choice(np.arange(1, n), size=P - 1, replace=False))
    return np.concatenate([[0], cuts, [n]]).astype(np.uint64)


@pytest.mark.parametrize("seed", range(6))
def test_invariants_random_partitions(seed):
    """For any partition: true start of C_k in I_sigma_k U Z,
    map_k[rank(start_k)] = start_{k+1}, fold = sequential final (Eq.SeqReduction,
    failure-freedom P:31-34)."""
    rng = np.random.default_rng(seed)
    makers = [lambda: automata.random_dfa(int(rng.integers(2, 40)), int(rng.integers(1, 9)), seed),
              lambda: automata.random_dfa_with_sink(int(rng.integers(3, 40)), int(rng.integers(1, 9)), seed),
              lambda: automata.random_structured(32, 16, 5, 8, seed)]
    for make in makers:
        aut = make()
        d = Dfa(aut.table, aut.q0, aut.accepting)
        n = int(rng.integers(50, 3000))
        x = rng.integers(0, aut.ns, n).astype(np.uint8)
        P = int(rng.integers(1, min(n, 40)))
        b = _random_partition(rng, n, P) if P > 1 else np.array([0, n], np.uint64)
        imax = max(d.imax(), 1)
        e0, maps = d.maps(x, b, imax)
        starts, fin = d.run_record(x, b[:-1])
        assert fin == d.run(x)
        assert d.fold(x, b, imax, e0, maps) == fin
        for k in range(1, P):
            I = d.initial_states(x[b[k] - 1]).tolist()
            s = int(starts[k])
            nxt = int(starts[k + 1]) if k + 1 < P else fin
            if d.dead[s]:
                assert nxt == s
                continue
            assert s in I
            assert maps[k - 1][I.index(s)] == nxt
        if P > 1:
            assert e0 == starts[1]


def test_p1_equals_sequential():
    aut = automata.random_dfa(20, 4, 3)
    d = Dfa(aut.table, aut.q0, aut.accepting)
    x = np.random.default_rng(0).integers(0, 4, 1000).astype(np.uint8)
    e0, maps = d.maps(x, np.array([0, x.size], np.uint64), d.imax())
    assert maps.shape[0] == 0 and e0 == d.run(x)


def test_compose_dense_paper_example(golden_dir):
    """Eq.MapReduction on Fig.motivDFA's dense chunk maps, derived by
    hand from the figure: L_{0,1,2}[q0] = q1 (accepted final P:243).
    The reversed operand order (L_i[L_j[q]]) gives qE and fails here."""
    g = load(golden_dir, "fig_motiv_dfa.json")
    L0, L1, L2 = (np.array(g[k], np.uint16) for k in ("L0_dense", "L1_dense", "L2_dense"))
    assert oracle.compose_dense(L0, L1).tolist() == g["L01_dense"]
    assert oracle.compose_dense(L1, L2).tolist() == g["L12_dense"]
    L012 = oracle.compose_dense(oracle.compose_dense(L0, L1), L2)
    assert L012.tolist() == g["L012_dense"]
    assert int(L012[g["q0"]]) == g["expected_final"]
    # the printed part of L2
    assert L2[[0, 1]].tolist() == g["L2_over_q0_q1"]


def test_compose_dense_is_concatenation():
    """Eq.MapReduction is the map of the concatenated chunk: with M(w)[q] =
    delta-hat(q, w) (Alg.seqmatch from every start state, pinned separately),
    compose_dense(M(u), M(v)) == M(uv) for random DFAs and strings.  A swapped
    operand order or an index slip fails on non-commuting maps."""
    rng = np.random.default_rng(4)
    for _ in range(40):
        nq, ns = int(rng.integers(2, 30)), int(rng.integers(1, 6))
        table = rng.integers(0, nq, (nq, ns)).astype(np.uint16)

        def M(w):
            return np.array([Dfa(table, q, []).run(w) for q in range(nq)], np.uint16)

        u = rng.integers(0, ns, int(rng.integers(0, 12))).astype(np.uint8)
        v = rng.integers(0, ns, int(rng.integers(0, 12))).astype(np.uint8)
        assert oracle.compose_dense(M(u), M(v)).tolist() == M(np.concatenate([u, v])).tolist()
        # associativity (a property the paper relies on for the binary reduction)
        A, B, C = (rng.integers(0, nq, nq).astype(np.uint16) for _ in range(3))
        assert (oracle.compose_dense(oracle.compose_dense(A, B), C).tolist()
                == oracle.compose_dense(A, oracle.compose_dense(B, C)).tolist())


def test_lemma1_containment():
    """Lemma 1, stronger form: I_{s' s} subset of I_s, hence
    I_max,r non-increasing in r (reading A15)."""
    for seed in range(4):
        aut = automata.random_structured(40, 6, 9, 10, seed)
        d = Dfa(aut.table, aut.q0, aut.accepting)
        imax_r = []
        for r in range(1, 4):
            best = 0
            for syms in itertools.product(range(6), repeat=r):
                I = set(d.initial_states_r(list(syms)).tolist())
                best = max(best, len(I))
                if r > 1:
                    assert I <= set(d.initial_states_r(list(syms[1:])).tolist())
            imax_r.append(best)
        assert imax_r[0] == d.imax()
        assert imax_r == sorted(imax_r, reverse=True)


def test_bounds_properties():
    """c-form properties that hold for any n >= c + P - 1."""
    rng = np.random.default_rng(7)
    for _ in range(300):
        P = int(rng.integers(1, 200))
        a, bb = int(rng.integers(1, 20)), int(rng.integers(1, 5))
        n = int(rng.integers(a // bb + P, 10 ** 7))
        b = oracle.chunk_bounds_ratio(n, P, a, bb).astype(np.int64)
        assert b[0] == 0 and b[-1] == n
        L = np.diff(b)
        assert (L >= 1).all()
        if P > 2:
            assert L[1:].max() - L[1:].min() <= 1
        if P > 1:
            # chunk 0 is c times the others up to rounding
            assert abs(L[0] * bb - a * L[1]) <= (a + 2 * bb) * 2


def test_bad_symbol_detected():
    d = Dfa(automata.counter_dfa(5, 4).table, 0, [0])
    with pytest.raises(oracle.OracleError):
        d.run(np.array([0, 1, 4], np.uint8))


# --------------------------------------------------------------------------- N1: r-symbol lookahead
def test_lookahead2_example_golden(golden_dir):
    """Eq.istatesm / Alg.TwoSymISet on Fig.ExampleDFA, values derived by hand
    in the fixture; chunk maps over I_{s1 s2} for the Fig.InputString split."""
    g = load(golden_dir, "fig_example_dfa.json")
    h = load(golden_dir, "fig_example_lookahead2.json")
    d = example_dfa(g)
    sym = g["symbols"]
    for w, want in h["I2"].items():
        assert d.initial_states_r([sym[c] for c in w]).tolist() == want
    assert max(len(v) for v in h["I2"].values()) == h["I_max_2"]
    x = enc(g["input"], sym)
    for ch in h["chunks_m2_r2"]:
        dom, row, cnt = d.chunk_map_r(x, ch["begin"], ch["end"], 2, 2)
        assert dom[:cnt].tolist() == ch["domain"] and row[:cnt].tolist() == ch["row"]
        assert (dom[cnt:] == 0xFFFF).all() and (row[cnt:] == 0xFFFF).all()


def test_chunk_map_r_properties():
    """r-symbol maps against brute force: the true state at every chunk start is
    in the r-domain (unless in Z) and its entry is the true state at the chunk
    end (sequential run); r = 1 is the I_sigma map; the r-domain shrinks with r
    (Lemma 1) and its rows are the I_sigma rows restricted (same delta-hat)."""
    rng = np.random.default_rng(11)
    for seed in range(6):
        aut = automata.random_structured(30, 5, 8, 6, seed) if seed % 2 else automata.random_dfa_with_sink(25, 4, seed)
        d = Dfa(aut.table, aut.q0, aut.accepting)
        dead = d.dead
        ns = aut.table.shape[1]
        x = rng.integers(0, ns, 400).astype(np.uint8)
        cuts = np.sort(rng.choice(np.arange(1, x.size), 12, replace=False))
        bounds = np.concatenate([[0], cuts, [x.size]])
        at, fin = d.run_record(x, bounds[:-1].astype(np.uint64))
        truth = at.tolist() + [fin]
        for k in range(1, bounds.size - 1):
            b, e = int(bounds[k]), int(bounds[k + 1])
            row1, c1 = d.chunk_map(x, b, e, d.nq)
            I1 = d.initial_states(int(x[b - 1])).tolist()
            prev = None
            for r in range(1, 6):
                dom, row, cnt = d.chunk_map_r(x, b, e, r, d.nq)
                D = dom[:cnt].tolist()
                if r == 1:
                    assert D == I1 and row[:cnt].tolist() == row1[:c1].tolist()
                if prev is not None:
                    assert set(D) <= set(prev)
                prev = D
                # brute force domain: the image of every state under the L symbols before b
                L = min(r, b)
                img = set()
                for q in range(d.nq):
                    s = q
                    for c in x[b - L:b]:
                        s = int(aut.table[s, c])
                    if not dead[s]:
                        img.add(s)
                assert D == sorted(img)
                for i, q in enumerate(D):
                    assert row[i] == row1[I1.index(q)]
                t = int(truth[k])
                if not dead[t]:
                    assert t in D
                    assert row[D.index(t)] == truth[k + 1]

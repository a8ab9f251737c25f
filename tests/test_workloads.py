"""Generator self-checks (-m "not gpu"): the synthetic workloads have the
structure DESIGN.md's input recipe states."""
import numpy as np

import workloads as W
from workloads import automata, inputs

APPENDIX_A = [[1, 2, 0, 0], [1, 3, 0, 0], [1, 2, 0, 4], [1, 2, 5, 4],
              [1, 2, 0, 6], [6, 2, 0, 0], [6, 6, 6, 6]]


def images(table):
    return [np.unique(table[:, c]).size for c in range(table.shape[1])]


def test_tiny_is_appendix_a():
    a = W.get("tiny").automaton
    assert a.table.tolist() == APPENDIX_A
    assert a.q0 == 0 and a.accepting.nonzero()[0].tolist() == [6]


def test_random_structured_images_exact():
    a = W.get("random").automaton
    assert a.nq == 64 and a.ns == 256 and a.accepting.sum() == 16
    assert set(images(a.table)) == {7}
    w = W.get("worst").automaton
    assert w.nq == 512 and w.accepting.sum() == 128
    assert set(images(w.table)) == {240}


def test_keyword_and_protein_shapes():
    k = W.get("keyword")
    assert 100 <= k.automaton.nq <= 400
    assert k.automaton.accepting.sum() == 1
    p = W.get("protein")
    assert 300 <= p.automaton.nq <= 1300
    # non-residue bytes go to one dead sink
    res = set(automata.RESIDUES)
    foreign = [b for b in range(256) if b not in res]
    assert np.unique(p.automaton.table[:, foreign]).size == 1


def test_inputs_deterministic_and_distributed():
    x1 = inputs.uniform_bytes(3 << 24, seed=1)
    x2 = inputs.uniform_bytes(3 << 24, seed=1)
    assert np.array_equal(x1, x2)
    assert not np.array_equal(x1[:1000], inputs.uniform_bytes(1000, seed=2))
    h = np.bincount(x1, minlength=256)
    assert h.min() > 0.95 * x1.size / 256
    r = inputs.uniform_over(automata.RESIDUES, 1 << 20, seed=0)
    assert set(np.unique(r).tolist()) == set(automata.RESIDUES)
    z = inputs.zipf_printable(1 << 22, seed=0)
    cnt = np.bincount(z, minlength=256)
    assert cnt[:0x20].sum() == 0 and cnt[0x7F:].sum() == 0
    p = cnt[0x20:0x7F] / z.size
    # rank 1 (space) ~0.2355, rank 2 ~0.1099
    assert abs(p[0] - 0.2355) < 0.003 and abs(p[1] - 0.1099) < 0.003


def test_planting():
    x = np.zeros(1 << 20, np.uint8)
    kws = [b"abcd", b"xyz12"]
    c = inputs.plant(x, kws, 1e-4, seed=0)
    assert 60 < c < 150
    s = bytes(x)
    assert s.count(b"abcd") + s.count(b"xyz12") >= c - 2

"""Seeded DFA constructions for the synthetic workloads.

These build the *inputs* of the method (a transition table, a start state and a
set of final states); they hold none of the method's arithmetic (no initial
state sets, no partitioning, no matching, no composition).  Both the CUDA path
and the oracle consume their output.

The paper builds minimal DFAs from PCRE / PROSITE patterns with Grail+
(P:1405-1409, 1667-1676).  Those corpora are not available, so the configs of
BASELINE.json are synthesised here: Aho-Corasick keyword DFAs (PCRE-style
multi-literal search), a PROSITE-style motif DFA, and random structured DFAs
whose per-symbol images have a fixed size (the paper's gamma range 0.02-0.47,
P:57).
"""
from __future__ import annotations

from collections import deque
from typing import Iterable, List, Sequence, Tuple

import numpy as np


class Automaton:
    """Plain container: table[q, c] = delta(q, c) over symbols 0..ns-1."""

    def __init__(self, table: np.ndarray, q0: int, accepting: np.ndarray, name: str = ""):
        self.table = np.ascontiguousarray(table, dtype=np.uint16)
        self.q0 = int(q0)
        self.accepting = np.asarray(accepting, dtype=bool)
        self.name = name
        assert self.table.ndim == 2 and self.accepting.shape == (self.table.shape[0],)

    @property
    def nq(self) -> int:
        return self.table.shape[0]

    @property
    def ns(self) -> int:
        return self.table.shape[1]

    @property
    def accept_bitmap(self) -> np.ndarray:
        bm = np.packbits(self.accepting, bitorder="little")
        return bm if bm.size else np.zeros(1, np.uint8)

    def digest(self) -> str:
        import hashlib
        h = hashlib.sha256()
        h.update(self.table.tobytes())
        h.update(np.int64(self.q0).tobytes())
        h.update(self.accept_bitmap.tobytes())
        return h.hexdigest()


# ---------------------------------------------------------------------------
# Minimisation (Moore partition refinement) + BFS renumbering from q0.
# ---------------------------------------------------------------------------
def reachable(table: np.ndarray, q0: int) -> np.ndarray:
    seen = np.zeros(table.shape[0], bool)
    seen[q0] = True
    frontier = [q0]
    while frontier:
        nxt = np.unique(table[frontier].ravel())
        new = nxt[~seen[nxt]]
        seen[new] = True
        frontier = new.tolist()
    return seen


def minimize(table: np.ndarray, q0: int, accepting: np.ndarray) -> Tuple[np.ndarray, int, np.ndarray]:
    table = np.asarray(table, dtype=np.int64)
    keep = np.nonzero(reachable(table, q0))[0]
    remap = -np.ones(table.shape[0], np.int64)
    remap[keep] = np.arange(keep.size)
    t = remap[table[keep]]
    acc = np.asarray(accepting, bool)[keep]
    q = int(remap[q0])
    cls = acc.astype(np.int64)
    ncls = np.unique(cls).size
    while True:
        sig = np.concatenate([cls[:, None], cls[t]], axis=1)
        _, new = np.unique(sig, axis=0, return_inverse=True)
        new = new.ravel()
        n_new = int(new.max()) + 1 if new.size else 0
        cls = new
        if n_new == ncls:
            break
        ncls = n_new
    # representative transitions per class
    rep = np.zeros(ncls, np.int64)
    rep[cls] = np.arange(cls.size)
    mt = cls[t[rep]]
    macc = acc[rep]
    mq0 = int(cls[q])
    # BFS renumbering from q0, symbols in increasing order
    order = -np.ones(ncls, np.int64)
    order[mq0] = 0
    nxt_id = 1
    dq = deque([mq0])
    while dq:
        s = dq.popleft()
        for c in range(mt.shape[1]):
            d = mt[s, c]
            if order[d] < 0:
                order[d] = nxt_id
                nxt_id += 1
                dq.append(d)
    inv = np.argsort(order)
    out = order[mt[inv]]
    return out.astype(np.uint16), 0, macc[inv]


# ---------------------------------------------------------------------------
# Aho-Corasick DFA for Sigma* (k_1 | ... | k_m) Sigma* with an absorbing ACC.
# ---------------------------------------------------------------------------
def aho_corasick(keywords: Sequence[Sequence[int]], ns: int) -> Automaton:
    goto: List[dict] = [dict()]
    out = [False]
    for kw in keywords:
        s = 0
        for c in kw:
            c = int(c)
            assert 0 <= c < ns
            if c not in goto[s]:
                goto.append(dict())
                out.append(False)
                goto[s][c] = len(goto) - 1
            s = goto[s][c]
        out[s] = True
    n = len(goto)
    fail = [0] * n
    table = np.zeros((n, ns), np.int64)
    dq = deque()
    for c in range(ns):
        if c in goto[0]:
            d = goto[0][c]
            table[0, c] = d
            fail[d] = 0
            dq.append(d)
        else:
            table[0, c] = 0
    while dq:
        s = dq.popleft()
        out[s] = out[s] or out[fail[s]]
        for c in range(ns):
            if c in goto[s]:
                d = goto[s][c]
                fail[d] = int(table[fail[s], c])
                table[s, c] = d
                dq.append(d)
            else:
                table[s, c] = table[fail[s], c]
    acc = np.array(out, bool)
    # merge all accepting nodes into one absorbing ACC state (Sigma* K Sigma*)
    acc_id = n
    table = np.concatenate([table, np.full((1, ns), acc_id, np.int64)], axis=0)
    acc = np.concatenate([acc, [True]])
    table[acc[:n].nonzero()[0]] = acc_id
    table = np.where(acc[table], acc_id, table)
    t, q0, a = minimize(table, 0, acc)
    return Automaton(t, q0, a, "aho-corasick")


# ---------------------------------------------------------------------------
# Random structured DFA: every symbol's image delta(Q, sigma) has exactly k
# states (surjective construction), delta(q, sigma) uniform within it.
# ---------------------------------------------------------------------------
def random_structured(nq: int, ns: int, k: int, n_accept: int, seed: int) -> Automaton:
    rng = np.random.Generator(np.random.Philox(key=(0xD5A << 40) ^ seed))
    table = np.zeros((nq, ns), np.uint16)
    for c in range(ns):
        image = rng.choice(nq, size=k, replace=False)
        perm = rng.permutation(nq)
        col = np.empty(nq, np.int64)
        col[perm[:k]] = image
        col[perm[k:]] = image[rng.integers(0, k, size=nq - k)]
        table[:, c] = col
    acc = np.zeros(nq, bool)
    acc[rng.choice(nq, size=n_accept, replace=False)] = True
    return Automaton(table, 0, acc, f"random(nq={nq},ns={ns},k={k})")


# ---------------------------------------------------------------------------
# PROSITE-style motif DFA: minimal DFA of Sigma* M Sigma* over 20 residues.
# ---------------------------------------------------------------------------
RESIDUES = b"ACDEFGHIKLMNPQRSTVWY"


def random_motif(rng: np.random.Generator, positions: int = 14):
    """Motif as a list of (kind, set_of_residue_indices, lo, hi)."""
    motif = []
    for _ in range(positions):
        u = rng.random()
        if u < 0.35:
            motif.append(("res", {int(rng.integers(20))}, 1, 1))
        elif u < 0.65:
            size = int(rng.integers(2, 6))
            motif.append(("class", set(rng.choice(20, size, replace=False).tolist()), 1, 1))
        elif u < 0.80:
            size = int(rng.integers(1, 4))
            excl = set(rng.choice(20, size, replace=False).tolist())
            motif.append(("excl", set(range(20)) - excl, 1, 1))
        else:
            motif.append(("gap", set(range(20)), 2, 4))
    return motif


def motif_text(motif) -> str:
    parts = []
    for kind, s, lo, hi in motif:
        letters = "".join(chr(RESIDUES[i]) for i in sorted(s))
        if kind == "res":
            parts.append(letters)
        elif kind == "class":
            parts.append("[" + letters + "]")
        elif kind == "excl":
            parts.append("{" + "".join(chr(RESIDUES[i]) for i in sorted(set(range(20)) - s)) + "}")
        else:
            parts.append(f"x({lo},{hi})")
    return "-".join(parts)


def _motif_slots(motif):
    slots = []  # (set, optional)
    for kind, s, lo, hi in motif:
        for _ in range(lo):
            slots.append((frozenset(s), False))
        for _ in range(hi - lo):
            slots.append((frozenset(s), True))
    return slots


def motif_dfa_residues(motif, max_states: int = 60000) -> Automaton | None:
    """Subset construction + minimisation over the 20-residue alphabet."""
    slots = _motif_slots(motif)
    L = len(slots)

    def closure(bits: int) -> int:
        # epsilon moves skip optional slots: i -> i+1 if slot i optional
        changed = True
        while changed:
            changed = False
            for i in range(L):
                if (bits >> i) & 1 and slots[i][1] and not (bits >> (i + 1)) & 1:
                    bits |= 1 << (i + 1)
                    changed = True
        return bits

    start = closure(1)
    ids = {start: 0}
    order = [start]
    rows = []
    i = 0
    while i < len(order):
        cur = order[i]
        row = []
        for c in range(20):
            nxt = 1  # Sigma* prefix: position 0 is always active
            if (cur >> L) & 1:
                nxt |= 1 << L  # Sigma* suffix: final position stays active
            for p in range(L):
                if (cur >> p) & 1 and c in slots[p][0]:
                    nxt |= 1 << (p + 1)
            nxt = closure(nxt)
            if nxt not in ids:
                ids[nxt] = len(order)
                order.append(nxt)
                if len(order) > max_states:
                    return None
            row.append(ids[nxt])
        rows.append(row)
        i += 1
    table = np.array(rows, np.int64)
    acc = np.array([(s >> L) & 1 == 1 for s in order], bool)
    t, q0, a = minimize(table, 0, acc)
    return Automaton(t, q0, a, "motif-residues")


def extend_to_bytes(aut: Automaton, alphabet: bytes) -> Automaton:
    """Byte-level table: byte alphabet[i] -> symbol i, every other byte -> a dead sink."""
    nq = aut.nq
    dead = nq
    table = np.full((nq + 1, 256), dead, np.uint16)
    for i, b in enumerate(alphabet):
        table[:nq, b] = aut.table[:, i]
    acc = np.concatenate([aut.accepting, [False]])
    return Automaton(table, aut.q0, acc, aut.name + "+bytes")


def protein_motif_dfa(seed: int, lo: int = 300, hi: int = 1300, positions: int = 14):
    """Resample seed, seed+1, ... until lo <= |Q| <= hi (reading A19). Returns (automaton, motif, seed_used)."""
    s = seed
    while True:
        rng = np.random.Generator(np.random.Philox(key=(0x9B07 << 40) ^ s))
        motif = random_motif(rng, positions)
        aut = motif_dfa_residues(motif)
        if aut is not None:
            full = extend_to_bytes(aut, RESIDUES)
            if lo <= full.nq <= hi:
                full.name = f"protein-motif {motif_text(motif)}"
                return full, motif, s
        s += 1


# ---------------------------------------------------------------------------
# Closed-form DFAs (pins P5).
# ---------------------------------------------------------------------------
def counter_dfa(nq: int, ns: int = 256) -> Automaton:
    """delta(q, c) = (q + c) mod |Q|: final = (q0 + sum bytes) mod |Q|."""
    q = np.arange(nq)[:, None]
    c = np.arange(ns)[None, :]
    return Automaton(((q + c) % nq).astype(np.uint16), 0, np.arange(nq) == 0, f"counter({nq})")


def reset_dfa(nq: int, f: np.ndarray) -> Automaton:
    """delta(q, c) = f(c): final = f(last byte)."""
    f = np.asarray(f, np.uint16)
    table = np.tile(f[None, :], (nq, 1))
    return Automaton(table, 0, np.arange(nq) % 2 == 1, "reset")


def identity_dfa(nq: int, ns: int = 256) -> Automaton:
    table = np.tile(np.arange(nq, dtype=np.uint16)[:, None], (1, ns))
    return Automaton(table, 0, np.arange(nq) == 0, "identity")


def permutation_dfa(nq: int, ns: int, seed: int) -> Automaton:
    """Every column a permutation of Q: maps are permutations, fold is a group product."""
    rng = np.random.Generator(np.random.Philox(key=(0x7E2 << 40) ^ seed))
    table = np.stack([rng.permutation(nq) for _ in range(ns)], axis=1).astype(np.uint16)
    return Automaton(table, 0, rng.random(nq) < 0.5, "permutation")


def random_dfa(nq: int, ns: int, seed: int, accept_frac: float = 0.3) -> Automaton:
    """Unstructured random DFA (fuzzing)."""
    rng = np.random.Generator(np.random.Philox(key=(0xF22 << 40) ^ seed))
    table = rng.integers(0, nq, size=(nq, ns)).astype(np.uint16)
    return Automaton(table, int(rng.integers(nq)), rng.random(nq) < accept_frac, "random")


def random_dfa_with_sink(nq: int, ns: int, seed: int, sink_frac: float = 0.3) -> Automaton:
    """Random DFA with an error state q_E (last state), reached with probability sink_frac."""
    rng = np.random.Generator(np.random.Philox(key=(0x51C << 40) ^ seed))
    table = rng.integers(0, nq - 1, size=(nq, ns))
    table[rng.random((nq, ns)) < sink_frac] = nq - 1
    table[nq - 1, :] = nq - 1
    acc = rng.random(nq) < 0.4
    acc[nq - 1] = False
    return Automaton(table.astype(np.uint16), 0, acc, "random+sink")

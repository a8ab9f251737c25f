"""Seeded synthetic workloads standing in for the paper's PCRE / PROSITE benchmarks.

The five configurations of BASELINE.json ("configs"), each as
(automaton, input generator, default chunk count P).
gives the recipe and the readings (A16-A20 of SURVEY.md section 8(c)).  The
paper's corpora (PCRE library, PROSITE) are not used: nothing here reproduces
any of their entries.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from typing import Callable, Dict, Optional

import numpy as np

from . import automata, inputs
from .automata import Automaton

MiB = 1 << 20
GiB = 1 << 30


@dataclass
class Workload:
    name: str
    automaton: Automaton
    alphabet_size: int
    full_n: int
    small_n: int
    chunks: int
    make_input: Callable[[int], np.ndarray]
    info: Dict = field(default_factory=dict)

    def input(self, n: Optional[int] = None, out=None, segment: int = 0) -> np.ndarray:
        """n input bytes; segment s > 0 draws an independent continuation (same
        automaton, input seed offset by s) -- segment s of a sharded input."""
        n = self.full_n if n is None else int(n)
        return self.make_input(n, out, segment)


def tiny(seed: int = 0) -> Workload:
    # Sigma*(abca|bdd)Sigma* over {a,b,c,d} = symbols 0..3 (Appendix A of SURVEY.md).
    aut = automata.aho_corasick([[0, 1, 2, 0], [1, 3, 3]], 4)
    aut.name = "tiny: AC(abca|bdd) over {a,b,c,d}"
    return Workload("tiny", aut, 4, 1 * MiB, 1 * MiB, 64,
                    lambda n, out=None, sg=0: inputs.uniform_over([0, 1, 2, 3], n, seed + 1000 * sg, out))


def random_structured(seed: int = 0) -> Workload:
    aut = automata.random_structured(64, 256, 7, 16, seed)
    return Workload("random", aut, 256, 256 * MiB, 4 * MiB, 4096,
                    lambda n, out=None, sg=0: inputs.uniform_bytes(n, seed + 1000 * sg, out))


def keyword(seed: int = 0) -> Workload:
    kws = inputs.random_keywords(32, seed)
    aut = automata.aho_corasick([list(k) for k in kws], 256)
    aut.name = "keyword: AC of 32 random printable keywords"

    def make(n, out=None, sg=0):
        x = inputs.zipf_printable(n, seed + 1000 * sg, 1.1, out)
        inputs.plant(x, kws, 1e-6, seed + 1000 * sg)
        return x

    return Workload("keyword", aut, 256, 1 * GiB, 4 * MiB, 16384, make,
                    {"keywords": [k.decode("latin1") for k in kws]})


def protein(seed: int = 0) -> Workload:
    aut, motif, used = automata.protein_motif_dfa(seed)
    return Workload("protein", aut, 256, 4 * GiB, 2 * MiB, 4096,
                    lambda n, out=None, sg=0: inputs.uniform_over(automata.RESIDUES, n, seed + 1000 * sg, out),
                    {"motif": automata.motif_text(motif), "motif_seed": used})


def worst(seed: int = 0) -> Workload:
    aut = automata.random_structured(512, 256, 240, 128, seed)
    return Workload("worst", aut, 256, 10 * GiB, 1 * MiB, 4096,
                    lambda n, out=None, sg=0: inputs.uniform_bytes(n, seed + 1000 * sg, out))


CONFIGS = {
    "tiny": tiny,
    "random": random_structured,
    "keyword": keyword,
    "protein": protein,
    "worst": worst,
}


def get(name: str, seed: int = 0) -> Workload:
    return CONFIGS[name](seed)


def sha256(x: np.ndarray) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(x))).hexdigest()

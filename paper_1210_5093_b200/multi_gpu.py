"""One input string sharded over G GPUs: the on-NVLink form of
the paper's two-tier merge (Fig.Merge).

Rank g holds segment g of x = x_0 x_1 ... x_{G-1} in its HBM.  It computes the
composed map of its segment over I_sigma of the previous segment's last byte
(one halo byte, exchanged once), the G rows (<= I_max uint16 each) are
all-gathered -- the only data-path collective -- and every rank folds them in
order (Eq.SeqReduction) into the replicated final state.

Orchestration only: the segment map and the fold are injected.  On GPUs they
are the library's kernels (``dfa_segment_map`` / ``dfa_fold_segments``, see
``gpu_ops``); the CPU tests inject the oracle to check this host logic under
``gloo`` with world size 2.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import torch


def exchange_halo(last_byte: torch.Tensor, dist, group=None) -> List[int]:
    """All-gather every segment's last byte; returns lookahead[g] = last byte of
    segment g-1 (-1 for segment 0: it starts from q0)."""
    world = dist.get_world_size(group)
    out = [torch.empty_like(last_byte) for _ in range(world)]
    dist.all_gather(out, last_byte, group=group)
    return [-1] + [int(t.reshape(-1)[0].item()) for t in out[:-1]]


def gather_rows(row: torch.Tensor, dist, group=None) -> torch.Tensor:
    """All-gather the uint16 segment rows (sent as bytes: NCCL has no 16-bit int type)."""
    world = dist.get_world_size(group)
    b = row.contiguous().view(torch.uint8)
    out = torch.empty(world * b.numel(), dtype=torch.uint8, device=b.device)
    dist.all_gather_into_tensor(out, b, group=group)
    return out.view(row.dtype).view(world, row.numel())


class SegmentMatcher:
    """Per-rank driver: step() = segment map, one all-gather, fold.  With one rank the
    segment is the whole string (lookahead -1): step() returns its map row, whose entry
    0 is the final state -- the same per-GPU work as every rank of a larger world."""

    def __init__(self, rank: int, world: int, dist, last_byte: torch.Tensor,
                 segment_map: Callable[[int], torch.Tensor],
                 fold: Callable[[torch.Tensor, List[int]], object], group=None):
        self.rank, self.world, self.dist, self.group = rank, world, dist, group
        self.lookahead = exchange_halo(last_byte, dist, group) if world > 1 else [-1]
        self.segment_map = segment_map
        self.fold = fold

    def step(self):
        row = self.segment_map(self.lookahead[self.rank])
        if self.world == 1:
            return row
        rows = gather_rows(row, self.dist, self.group)
        return self.fold(rows, self.lookahead)


def gpu_ops(d, dev_input: torch.Tensor, stream=None, chunks: int = 1):
    """(segment_map, fold) for a D.Dfa handle on this rank's segment, all in the
    library's kernels; results stay on the device (fold returns {final, accept}).
    segment_map runs dfa_segment_chunk_maps with `chunks` reporting chunks -- the same
    partition and kernels as dfa_chunk_maps on one GPU; its buffers are attributes
    (segment_map.bounds / .chunk0 / .maps / .row)."""
    import paper_1210_5093_b200 as D
    dev = dev_input.device
    imax = d.info["i_max"]
    P = int(chunks)
    row = torch.empty(imax, dtype=torch.int16, device=dev)
    bounds = torch.empty(P + 1, dtype=torch.int64, device=dev)
    chunk0 = torch.empty(imax, dtype=torch.int16, device=dev)
    maps = torch.empty(max(P - 1, 1) * imax, dtype=torch.int16, device=dev)
    final = torch.empty(2, dtype=torch.int16, device=dev)
    la_dev: Optional[torch.Tensor] = None

    def segment_map(lookahead: int) -> torch.Tensor:
        D.dfa_segment_chunk_maps(d.h, dev_input, P, lookahead, bounds, chunk0, maps, row, stream=stream)
        return row

    segment_map.bounds, segment_map.chunk0, segment_map.maps, segment_map.row = bounds, chunk0, maps, row

    def fold(rows: torch.Tensor, lookahead: List[int]):
        nonlocal la_dev
        if la_dev is None:
            la_dev = torch.tensor([max(v, 0) for v in lookahead], dtype=torch.uint8, device=dev)
        D.dfa_fold_segments(d.h, rows, la_dev, len(lookahead), final, stream=stream)
        return final

    return segment_map, fold

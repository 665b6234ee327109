"""Stage-level codebook construction on the GPU (huffman.py:79-180 of the reference).

``build_codebooks`` runs the same warp-per-histogram kernel (k_codebook +
k_pkgmerge) that the compressor uses for every block, on arbitrary
histograms: two-queue Huffman with leaf-first ties, and the package-merge
fallback with the reference's tie rules when a code would exceed 15 bits.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import EmptyInputError

MAX_CODE_LENGTH = 15


@dataclass(frozen=True)
class BlockCodebook:
    """256 code lengths in bits; 0 marks an absent symbol (huffman.py:46-61)."""

    lengths: np.ndarray

    @property
    def present(self) -> np.ndarray:
        return np.flatnonzero(self.lengths)

    def kraft_units(self) -> int:
        lens = self.lengths[self.lengths > 0].astype(np.int64)
        return int(np.sum(1 << (MAX_CODE_LENGTH - lens)))


def build_codebooks(hists) -> np.ndarray:
    """[N, 256] counts -> [N, 256] uint8 code lengths, computed on the GPU."""
    import torch

    h = np.ascontiguousarray(np.asarray(hists, dtype=np.int64))
    if h.ndim == 1:
        h = h[None]
    if h.shape[1] != 256:
        raise ValueError("histograms must have 256 bins")
    if h.size and (h.min() < 0 or h.sum(axis=1).max() >= (1 << 32)):
        raise ValueError("counts must be non-negative with totals below 2**32")
    ctx = _lib.context()
    dev = torch.device("cuda", ctx.device)
    dh = torch.from_numpy(h.astype(np.uint32).view(np.int32)).to(dev)
    dl = torch.zeros((h.shape[0], 256), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    rc = ctx.lib.lmcg_build_codebooks(ctx.ptr, dh.data_ptr(), h.shape[0], dl.data_ptr(), s.cuda_stream)
    if rc and rc != 6:
        ctx.check(rc)
    return dl.cpu().numpy()


def build_codebook(h) -> BlockCodebook:
    """Single-histogram form of the reference's ``build_codebook``."""
    counts = np.asarray(getattr(h, "counts", h), dtype=np.int64)
    if counts.sum() == 0:
        raise EmptyInputError("cannot build a codebook from an empty histogram")
    return BlockCodebook(build_codebooks(counts[None])[0])

"""Observation-sequence input for the B200 core: the reference's delimited
text format, parsed straight into one pinned host buffer and moved to the
device as a packed batch.

``read_sequences`` restates model_io.py:150-195 (same blocks, header rule,
column selection, error texts) and returns the reference's list of arrays;
``read_sequences_batch`` returns the same sequences as an ``engine.Batch``
instead: the values are written once into a growing page-locked buffer
(no per-sequence arrays, no concatenation copy), the CSR offsets are kept
alongside (the ``np.concatenate(seqs)`` layout of training.py:172), and the
buffer is copied to the GPU with one asynchronous host-to-device transfer on
the current stream.  Text is streamed in chunks, so a file larger than host
memory's comfort zone is never held as one string.
"""

from __future__ import annotations

import io
import math
from pathlib import Path

import numpy as np
import torch

from . import engine

__all__ = ["read_sequences", "read_sequences_batch"]

_CHUNK_LINES = 1 << 16


class _Packer:
    """Growing pinned float64 buffer + offsets."""

    def __init__(self, pinned: bool):
        self.pinned = pinned and torch.cuda.is_available()
        self.buf = self._alloc(1 << 16)
        self.n = 0
        self.offsets = [0]

    def _alloc(self, n):
        t = torch.empty(n, dtype=torch.float64)
        return t.pin_memory() if self.pinned else t

    def push(self, vals: list) -> None:
        m = len(vals)
        if self.n + m > self.buf.numel():
            nb = self._alloc(max(2 * self.buf.numel(), self.n + m))
            nb[: self.n] = self.buf[: self.n]
            self.buf = nb
        self.buf[self.n:self.n + m] = torch.tensor(vals, dtype=torch.float64)
        self.n += m

    def end_block(self) -> None:
        if self.n > self.offsets[-1]:
            self.offsets.append(self.n)


def _parse(source, column: int, delimiter: str, sink) -> None:
    """model_io.py:150-195 line by line; sink(values) per parsed chunk of a
    block, sink(None) at each block end."""
    if isinstance(source, (str, Path)):
        try:
            fh = open(source, encoding="utf-8")
        except OSError as exc:
            raise OSError(f"could not read sequences from {source}: {exc}") from exc
        close = True
    else:
        fh = source if not isinstance(source, (bytes, bytearray)) else io.StringIO(source.decode())
        close = False
    seen_data_row = False
    in_block = False
    pending: list[float] = []
    def logical_lines():
        # the reference splits the whole text with str.splitlines(); split
        # each physical line the same way so the numbering agrees
        for raw in fh:
            for sub in raw.splitlines() or [""]:
                yield sub

    try:
        for lineno, raw in enumerate(logical_lines(), start=1):
            line = raw.strip()
            if not line:
                if in_block:
                    sink(pending)
                    pending = []
                    sink(None)
                    in_block = False
                continue
            cells = line.split(delimiter)
            if column >= len(cells):
                raise ValueError(f"line {lineno}: row has {len(cells)} column(s), need column {column}")
            cell = cells[column].strip()
            try:
                value = float(cell)
            except ValueError:
                if not seen_data_row:
                    continue  # header row
                raise ValueError(f"line {lineno}: could not parse {cell!r} as a number") from None
            if math.isnan(value):
                raise ValueError(f"line {lineno}: NaN observation")
            seen_data_row = True
            in_block = True
            pending.append(value)
            if len(pending) >= _CHUNK_LINES:
                sink(pending)
                pending = []
        if in_block:
            sink(pending)
            sink(None)
    finally:
        if close:
            fh.close()


def read_sequences(source, column: int = 0, delimiter: str = ",") -> list[np.ndarray]:
    """Blank-line-delimited sequences from delimited text (model_io.py:150-195)."""
    seqs: list[np.ndarray] = []
    cur: list[float] = []

    def sink(vals):
        if vals is None:
            seqs.append(np.array(cur))
            cur.clear()
        else:
            cur.extend(vals)

    _parse(source, column, delimiter, sink)
    if not seqs:
        raise ValueError("no observation sequences found in input")
    return seqs


def read_sequences_batch(source, column: int = 0, delimiter: str = ",", dtype="float64",
                         device=None) -> engine.Batch:
    """The sequences of ``source`` as a device batch: parsed into one pinned
    buffer, one asynchronous H2D copy on the current stream."""
    pk = _Packer(pinned=True)

    def sink(vals):
        if vals is None:
            pk.end_block()
        elif vals:
            pk.push(vals)

    _parse(source, column, delimiter, sink)
    if len(pk.offsets) < 2:
        raise ValueError("no observation sequences found in input")
    dev = device or engine._device()
    td = engine.torch_dtype(dtype)
    host = pk.buf[: pk.n]
    y0 = host.to(device=dev, non_blocking=True).to(td)
    off = np.asarray(pk.offsets, dtype=np.int64)
    return engine.Batch(y0=y0.contiguous(), y1=None, offsets=torch.from_numpy(off).to(dev),
                        offsets_host=off, dtype=td)

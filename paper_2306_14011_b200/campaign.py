"""Long sweeps in checkpointed chunks: the paper's full space.

The paper's own search space has 10^7 x 12^7 = 3.58e14 configurations
(PAPER.md:241), which it could only sample.  Swept exhaustively at ~3.5e10
evals/s per B200 it takes ~1.3e3 s on 8 GPUs, long enough that a sweep must
survive interruption.  A campaign splits the index range [begin, end) into
chunks, sweeps each chunk to its k best records (K1 + K2 on the device), folds
them into the running top-k with the merge kernel, and every `every` chunks
writes the running records plus the next chunk's start to a checkpoint file
(atomic rename).  A new Campaign on the same file resumes after the last
checkpointed chunk.  Because the (t, idx) order is total and the merge is
exact, the result is bitwise identical to a one-shot sweep of the range,
whatever the chunking or the interruption points (tested).

Records are surr_record rows as int64 [k, 2] tensors (idx, key | pad << 32),
key = the kernels' order-preserving float -> uint32 map of t; sentinel rows
(idx = -1) pad short ranges.  Host logic only: every chunk runs in the CUDA
kernels through the binding.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

SENTINEL_IDX = -1
SENTINEL_KEY = 0xFFFFFFFF


def fingerprint(value_lists, k: int, begin: int, end: int, tag: str = "") -> str:
    """Identity of a campaign: space, range, k and a caller tag (model / precision)."""
    blob = json.dumps({"values": [[float(x) for x in v] for v in value_lists], "k": int(k),
                       "begin": int(begin), "end": int(end), "tag": str(tag)}, sort_keys=True)
    return hashlib.sha256(blob.encode()).hexdigest()


class Campaign:
    """Top-k of [begin, end) in chunks of `chunk` configs, resumable from `path`.

    local_sweep(lo, hi, k) -> [k, 2] int64 records of [lo, hi) (sorted, sentinel padded)
    merge(records [2k, 2], lists=2, k) -> [k, 2] merged records
    Both run on the device in the product path (`for_surrogate`)."""

    def __init__(self, local_sweep, merge, k: int, begin: int, end: int, chunk: int, path: str | None = None,
                 every: int = 1, fp: str = "", to_numpy=None, from_numpy=None):
        if not (0 <= begin <= end) or chunk < 1 or k < 1 or every < 1:
            raise ValueError("bad campaign range / chunk / k / every")
        self.local_sweep, self.merge = local_sweep, merge
        self.k, self.begin, self.end, self.chunk, self.every = int(k), int(begin), int(end), int(chunk), int(every)
        self.path, self.fp = path, fp
        self.to_numpy = to_numpy or (lambda r: r if isinstance(r, np.ndarray) else r.cpu().numpy())
        self.from_numpy = from_numpy
        self.next = self.begin
        self.recs = None          # running top-k records (None before the first chunk)
        self.chunks_done = 0      # chunks swept by this object (not counting resumed ones)
        self.resumed_from = None
        if path and os.path.exists(path):
            self._load()

    # ---------------------------------------------------------- checkpoint
    def _meta(self):
        return {"fp": self.fp, "k": self.k, "begin": self.begin, "end": self.end, "chunk": self.chunk}

    def _load(self):
        z = np.load(self.path, allow_pickle=False)
        meta = json.loads(str(z["meta"]))
        if meta != self._meta():
            raise ValueError(f"checkpoint {self.path} belongs to another campaign: {meta}")
        self.next = int(z["next"])
        if not (self.begin <= self.next <= self.end):
            raise ValueError("checkpoint position outside the campaign range")
        if int(z["has_recs"]):
            recs = np.asarray(z["recs"], np.int64)
            self.recs = self.from_numpy(recs) if self.from_numpy else recs
        self.resumed_from = self.next

    def save(self):
        if not self.path:
            return
        recs = self.to_numpy(self.recs) if self.recs is not None else np.zeros((self.k, 2), np.int64)
        tmp = self.path + ".tmp.npz"
        np.savez(tmp, meta=json.dumps(self._meta()), next=np.int64(self.next),
                 has_recs=np.int64(self.recs is not None), recs=np.asarray(recs, np.int64))
        os.replace(tmp, self.path)

    # ---------------------------------------------------------- sweep
    @property
    def finished(self) -> bool:
        return self.next >= self.end

    def step(self):
        """Sweep one chunk and fold it into the running top-k."""
        lo = self.next
        hi = min(lo + self.chunk, self.end)
        new = self.local_sweep(lo, hi, self.k)
        self.recs = new if self.recs is None else self.merge(_cat(self.recs, new), 2, self.k)
        self.next = hi
        self.chunks_done += 1
        if self.chunks_done % self.every == 0 or self.finished:
            self.save()

    def run(self, max_chunks: int | None = None):
        """Sweep until the range is done (or max_chunks chunks, to bound a session).
        Returns the running [k, 2] records (final once `finished`)."""
        n = 0
        while not self.finished and (max_chunks is None or n < max_chunks):
            self.step()
            n += 1
        if self.recs is None:  # empty range
            recs = np.zeros((self.k, 2), np.int64)
            recs[:, 0] = SENTINEL_IDX
            recs[:, 1] = SENTINEL_KEY
            self.recs = self.from_numpy(recs) if self.from_numpy else recs
        return self.recs


def _cat(a, b):
    if isinstance(a, np.ndarray):
        return np.concatenate([a, b])
    import torch
    return torch.cat([a, b])


def records_to_result(recs: np.ndarray, count: int):
    """[k, 2] int64 records -> (idx uint64 [count], t float32 [count])."""
    from . import key_to_float
    r = np.asarray(recs, np.int64)[:count]
    return r[:, 0].astype(np.uint64), key_to_float((r[:, 1] & 0xFFFFFFFF).astype(np.uint32))


def for_surrogate(surrogate, value_lists, k: int, begin: int, end: int, chunk: int, path: str | None = None,
                  every: int = 1, tag: str = "") -> Campaign:
    """The product campaign: chunks run K1 + K2 (`sweep_records`), folds run K2
    (`merge_topk`), records stay on the device between chunks."""
    import torch
    dev = f"cuda:{surrogate.device}"

    def local(lo, hi, kk):
        return surrogate.sweep_records(value_lists, kk, lo, hi)

    def merge(recs, lists, kk):
        return surrogate.merge_topk(recs, lists, kk, kk)[2]

    # the loaded model's digest is part of the identity: a checkpoint written
    # under other weights / precision is refused, not silently resumed
    tag = f"{tag}|model:{getattr(surrogate, 'model_digest', '')}"
    return Campaign(local, merge, k, begin, end, chunk, path, every, fingerprint(value_lists, k, begin, end, tag),
                    from_numpy=lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev))

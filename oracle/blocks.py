"""Deterministic block-allocator model (oracle of the device K6 allocator).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). No reference counterpart:
block tables are a reference non-goal; this model is the
contract the device allocator is checked against bit for bit.

* The free list is a LIFO stack, initialised so the first pops return
  blocks 0, 1, 2, ... .
* A batched allocation pops in batch order: request 0's logical blocks
  0..c0-1, then request 1's, ... (device: an exclusive scan of per-request
  block counts against the stack pointer).
* Frees push in request order, and within a request in ascending logical
  block order (device: scan of per-request free counts).
* Compaction keeps logical blocks [0, ceil(K_r / bs)) and frees the tail in
  the same batch step (pooled mode). Legacy mode pops fresh blocks for the
  compressed copy in batch order and keeps the raw blocks until release;
  release pushes the live blocks, then the retained raw blocks.
"""

from __future__ import annotations


def blocks_for(tokens: int, block_size: int) -> int:
    return -(-int(tokens) // block_size)


class BlockAllocatorModel:
    def __init__(self, num_blocks: int, block_size: int):
        self.block_size = block_size
        self.stack = list(range(num_blocks - 1, -1, -1))
        self.tables: dict[int, list[int]] = {}
        self.retained: dict[int, list[int]] = {}
        self.tokens: dict[int, int] = {}

    @property
    def free_blocks(self) -> int:
        return len(self.stack)

    def _pop(self, n: int) -> list[int]:
        if n > len(self.stack):
            raise RuntimeError("block pool exhausted")
        return [self.stack.pop() for _ in range(n)]

    def alloc_batch(self, handle_ids, tokens) -> None:
        for h, t in zip(handle_ids, tokens):
            self.tables[h] = self._pop(blocks_for(t, self.block_size))
            self.tokens[h] = int(t)

    def compress_batch(self, handle_ids, kept_tokens, legacy: bool = False) -> None:
        if legacy:
            for h, k in zip(handle_ids, kept_tokens):
                self.retained[h] = self.tables[h]
                self.tables[h] = self._pop(blocks_for(k, self.block_size))
                self.tokens[h] = int(k)
            return
        for h, k in zip(handle_ids, kept_tokens):
            keep = blocks_for(k, self.block_size)
            self.stack.extend(self.tables[h][keep:])
            del self.tables[h][keep:]
            self.tokens[h] = int(k)

    def append_batch(self, handle_ids, counts) -> None:
        for h, c in zip(handle_ids, counts):
            t = self.tokens[h]
            need = blocks_for(t + c, self.block_size) - blocks_for(t, self.block_size)
            self.tables[h].extend(self._pop(need))
            self.tokens[h] = t + int(c)

    def release_batch(self, handle_ids) -> None:
        for h in handle_ids:
            self.stack.extend(self.tables.pop(h))
            self.stack.extend(self.retained.pop(h, []))
            self.tokens.pop(h)

"""Ragged device arena: per-request state regions inside one HBM tensor.

Every live request owns a handful of variable-length regions (encoder
memory, two ping-pong decoder-state buffers, two vocoder-state buffers).
They are carved out of a single growable torch tensor by a best-fit
allocator with coalescing (free blocks indexed by start for coalescing and by
(size, start) for an O(log n) fit), so kernels address them with plain
base+offset pointers and no per-request cudaMalloc ever happens on the serving
path.

Offsets are in elements and 128-byte aligned.  Growth reallocates and
copies on the owning stream; callers keep offsets (never raw pointers)
across calls and rebuild pointers from :attr:`base_ptr` per call.
"""

from __future__ import annotations

import bisect
import collections
import threading

import torch

_ALIGN_BYTES = 128


class RaggedArena:
    def __init__(self, dtype: torch.dtype, device: torch.device, capacity: int, stream=None):
        self.dtype = dtype
        self.device = device
        self.itemsize = torch.tensor([], dtype=dtype).element_size()
        self.align = max(1, _ALIGN_BYTES // self.itemsize)
        self.stream = stream
        self._lock = threading.Lock()
        # frees from weakref finalizers: those can run inside a cyclic collection on ANY thread,
        # including this one while alloc() holds the lock, so they only append here (atomic, no
        # lock, no allocation-triggered re-entry) and the owning thread's next alloc() applies them
        self._deferred: collections.deque = collections.deque()
        cap = self._round(capacity)
        self.tensor = torch.empty(cap, dtype=dtype, device=device)
        self._free_starts = [0]
        self._free_sizes = {0: cap}
        self._by_size = [(cap, 0)]   # sorted (size, start) of the free blocks
        self._used = 0
        self.peak = 0

    def _round(self, n: int) -> int:
        return max(self.align, -(-int(n) // self.align) * self.align)

    @property
    def used(self) -> int:
        """Elements in use (queued finalizer frees applied first)."""
        self.drain()
        return self._used

    @property
    def capacity(self) -> int:
        return self.tensor.numel()

    @property
    def base_ptr(self) -> int:
        return self.tensor.data_ptr()

    def ptr(self, off: int) -> int:
        return self.tensor.data_ptr() + off * self.itemsize

    def release(self, off: int, n: int) -> None:
        """Finalizer-safe free: queued, applied by the next alloc() / free() / drain()."""
        self._deferred.append((off, n))

    def drain(self) -> None:
        with self._lock:
            self._drain_locked()

    def _drain_locked(self) -> None:
        while True:
            try:
                off, n = self._deferred.popleft()
            except IndexError:
                return
            size = self._round(n)
            self._used -= size
            self._insert_free(off, size)

    def alloc(self, n: int) -> int:
        size = self._round(n)
        with self._lock:
            self._drain_locked()
            j = bisect.bisect_left(self._by_size, (size, -1))   # smallest block that fits
            if j < len(self._by_size):
                have, start = self._by_size[j]
                self._remove_free(start, have, j)
                if have > size:
                    self._insert_free(start + size, have - size)
                self._used += size
                self.peak = max(self.peak, self._used)
                return start
            self._grow(size)
        return self.alloc(n)

    def _remove_free(self, start: int, size: int, j: int | None = None) -> None:
        del self._free_sizes[start]
        self._free_starts.pop(bisect.bisect_left(self._free_starts, start))
        if j is None:
            j = bisect.bisect_left(self._by_size, (size, start))
        self._by_size.pop(j)

    def free(self, off: int, n: int) -> None:
        size = self._round(n)
        with self._lock:
            self._drain_locked()
            self._used -= size
            self._insert_free(off, size)

    def _insert_free(self, start: int, size: int) -> None:
        i = bisect.bisect_left(self._free_starts, start)
        # coalesce with right neighbour
        if i < len(self._free_starts) and start + size == self._free_starts[i]:
            right = self._free_starts[i]
            rsize = self._free_sizes[right]
            self._remove_free(right, rsize)
            size += rsize
        # coalesce with left neighbour
        if i > 0:
            left = self._free_starts[i - 1]
            lsize = self._free_sizes[left]
            if left + lsize == start:
                self._remove_free(left, lsize)
                start, size = left, lsize + size
                i -= 1
        self._free_starts.insert(i, start)
        self._free_sizes[start] = size
        bisect.insort(self._by_size, (size, start))

    def _grow(self, need: int) -> None:
        old = self.tensor
        cap = old.numel()
        new_cap = self._round(max(2 * cap, cap + need))
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _nullctx()
        with ctx:
            new = torch.empty(new_cap, dtype=self.dtype, device=self.device)
            new[:cap].copy_(old)
        self.tensor = new
        self._insert_free(cap, new_cap - cap)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False

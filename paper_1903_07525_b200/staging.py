"""Host <-> HBM staging for the reference-compatible host API.

``PlanRunner.run`` takes and returns plain numpy arrays (executor.py:168-198),
so every call moves the input volume host -> device and the result back.
A single-threaded numpy copy into pinned memory runs at ~5-10 GB/s and would
dominate the end-to-end time, so transfers are chunked: a thread pool copies
chunk k into a pinned staging buffer (numpy releases the GIL) while the
copy engine moves chunk k-1 over PCIe, and on the way back chunk k is
unpacked into the fresh output array while chunk k+1 is still in flight.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK_BYTES = 4 << 20


def _workers() -> int:
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 4
    return max(2, min(16, n))


_POOL = None


def pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=_workers())
    return _POOL


def _spans(nbytes: int, chunk: int):
    return [(o, min(chunk, nbytes - o)) for o in range(0, nbytes, chunk)]


def _par_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (one chunk; chunks run concurrently on the pool)."""
    dst[:] = src


def pinned_empty(shape) -> np.ndarray:
    """Page-locked float32 host array: ``upload``/``download`` move it with one
    DMA each way, skipping the staging copy."""
    import torch
    return torch.empty(tuple(shape), dtype=torch.float32, pin_memory=True).numpy()


def is_pinned(a: np.ndarray) -> bool:
    import torch
    return (isinstance(a, np.ndarray) and not isinstance(a, np.memmap) and
            a.dtype == np.float32 and a.flags.c_contiguous and a.flags.writeable
            and torch.from_numpy(a).is_pinned())


def upload(host: np.ndarray, pinned, device_tensor, stream) -> None:
    """host (any float32-convertible array) -> device_tensor via pinned chunks
    (a page-locked float32 array goes in one DMA)."""
    import torch
    if is_pinned(host):
        with torch.cuda.stream(stream):
            device_tensor.copy_(torch.from_numpy(host), non_blocking=True)
        return
    src = np.ascontiguousarray(host, dtype=np.float32).reshape(-1).view(np.uint8)
    stage = pinned.reshape(-1).view(torch.uint8)
    stage_np = stage.numpy()
    dst = device_tensor.reshape(-1).view(torch.uint8)
    spans = _spans(src.size, CHUNK_BYTES)
    futs = [pool().submit(_par_copy, stage_np[o:o + n], src[o:o + n]) for o, n in spans]
    with torch.cuda.stream(stream):
        for (o, n), f in zip(spans, futs):
            f.result()
            dst[o:o + n].copy_(stage[o:o + n], non_blocking=True)


def download(device_tensor, pinned, stream, out=None) -> np.ndarray:
    """device_tensor -> host float32 array via pinned chunks; ``out`` (a
    page-locked array from ``pinned_empty``) receives it in one DMA."""
    import torch
    if out is not None:
        if tuple(out.shape) != tuple(device_tensor.shape) or not is_pinned(out):
            from .errors import ExecutionError
            raise ExecutionError("out= must be a pinned float32 array of shape %s"
                                 % (tuple(device_tensor.shape),))
        with torch.cuda.stream(stream):
            torch.from_numpy(out).copy_(device_tensor, non_blocking=True)
        stream.synchronize()
        return out
    src = device_tensor.reshape(-1).view(torch.uint8)
    stage = pinned.reshape(-1).view(torch.uint8)
    stage_np = stage.numpy()
    out = np.empty(tuple(device_tensor.shape), dtype=np.float32)
    out_b = out.reshape(-1).view(np.uint8)
    spans = _spans(out_b.size, CHUNK_BYTES)
    events = []
    with torch.cuda.stream(stream):
        for o, n in spans:
            stage[o:o + n].copy_(src[o:o + n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            events.append(ev)
    futs = []
    for (o, n), ev in zip(spans, events):
        ev.synchronize()
        futs.append(pool().submit(_par_copy, out_b[o:o + n], stage_np[o:o + n]))
    for f in futs:
        f.result()
    return out


# ------------------------------------------------------------------ row staging
# DeviceTiler.run_host streams a large volume row by row.  Page-locked host
# arrays move by direct DMA; pageable ones go through two pinned staging
# slots per direction, filled / drained by the thread pool while the copy
# engines and the convolutions work on the neighbouring rows.

def _plane_jobs(dst: np.ndarray, src: np.ndarray):
    """(dst, src) pairs of (b, c, x-block) sub-blocks of about CHUNK_BYTES."""
    nb, nc, nx = dst.shape[:3]
    plane = max(1, int(np.prod(dst.shape[3:])) * 4)
    step = max(1, CHUNK_BYTES // plane)
    return [(dst[b, c, x:x + step], src[b, c, x:x + step])
            for b in range(nb) for c in range(nc) for x in range(0, nx, step)]


class RowStager:
    """Two pinned staging slots per direction for pageable volumes."""

    def __init__(self):
        self._in = [None, None]      # (pinned tensor, DMA-done event)
        self._out = [None, None]     # (pinned tensor, host-copy future)

    @staticmethod
    def _grow(entry, numel):
        import torch
        if entry is None or entry[0].numel() < numel:
            return torch.empty(numel, dtype=torch.float32, pin_memory=True)
        return entry[0]

    def upload(self, slot, src_view: np.ndarray, dst, stream) -> None:
        """dst (contiguous device tensor) <- src_view (any host float32 view)."""
        import torch
        ent = self._in[slot]
        if ent is not None and ent[1] is not None:
            ent[1].synchronize()                 # the slot's previous DMA has read it
        buf = self._grow(ent, dst.numel())
        st = buf[:dst.numel()].view(dst.shape)
        st_np = st.numpy()
        futs = [pool().submit(np.copyto, d, s) for d, s in _plane_jobs(st_np, src_view)]
        for f in futs:
            f.result()
        with torch.cuda.stream(stream):
            dst.copy_(st, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        self._in[slot] = (buf, ev)

    def download(self, slot, src, out_view: np.ndarray, stream) -> None:
        """out_view (host view) <- src (contiguous device tensor), asynchronously:
        the DMA is enqueued on ``stream``, a pool thread copies the staged
        result into out_view once it lands (``finish`` waits for all)."""
        import torch
        ent = self._out[slot]
        if ent is not None and ent[1] is not None:
            ent[1].result()                      # the slot's previous host copy is done
        buf = self._grow(ent, src.numel())
        st = buf[:src.numel()].view(src.shape)
        with torch.cuda.stream(stream):
            st.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        st_np = st.numpy()

        def land():
            ev.synchronize()
            jobs = _plane_jobs(out_view, st_np)
            half = len(jobs) // 2
            # the other half in a second pool thread (at most two rows land
            # at once, so the pool never waits on itself)
            f = pool().submit(lambda: [np.copyto(d, s) for d, s in jobs[half:]])
            for d, s in jobs[:half]:
                np.copyto(d, s)
            f.result()
        self._out[slot] = (buf, pool().submit(land))

    def finish(self) -> None:
        for ent in self._out:
            if ent is not None and ent[1] is not None:
                ent[1].result()

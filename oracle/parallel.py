"""Throughput of the oracle AS IT STANDS on every host core (bench.py's cpu_baseline
and --impl reference legs; "the oracle runs on all host cores").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Nothing here changes the
oracle's arithmetic: independent worker processes (spawned, one per core) each
run oracle.extract_fingerprint on a slice of the same frames for a time budget;
throughput = all denoisings / wall time."""
from __future__ import annotations

import multiprocessing as mp
import os
import time
from multiprocessing import shared_memory

import numpy as np

_FR = None


def _init(name: str, shape):
    global _FR, _SHM
    _SHM = shared_memory.SharedMemory(name=name)
    _FR = np.ndarray(shape, dtype=np.uint8, buffer=_SHM.buf)


def _work(args):
    import oracle
    depth, start, budget = args
    n, t0 = 0, time.perf_counter()
    while True:
        oracle.extract_fingerprint(_FR[start:start + depth], depth)   # one SDA group = one denoising
        n += 1
        if time.perf_counter() - t0 >= budget:
            break
    return n


def sample(frames: np.ndarray, depths, budget_s: float, workers: int | None = None):
    """Denoisings/s of the oracle over `workers` processes (default: all cores) and a description."""
    workers = workers or os.cpu_count() or 1
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    shm = shared_memory.SharedMemory(create=True, size=frames.nbytes)
    try:
        np.ndarray(frames.shape, dtype=np.uint8, buffer=shm.buf)[:] = frames
        ctx = mp.get_context("spawn")
        total_n, total_t, desc = 0, 0.0, []
        with ctx.Pool(workers, initializer=_init, initargs=(shm.name, frames.shape)) as pool:
            pool.map(_work, [(1, 0, 0.0)] * workers)   # warm the workers (imports, library load)
            for d in depths:
                groups = max(1, frames.shape[0] // d)
                jobs = [(d, (w % groups) * d, budget_s / len(depths)) for w in range(workers)]
                t0 = time.perf_counter()
                n = sum(pool.map(_work, jobs))
                dt = time.perf_counter() - t0
                total_n += n
                total_t += dt
                desc.append(f"d={d}: {n} denoisings over {dt:.1f}s")
        return total_n / total_t, workers, "; ".join(desc)
    finally:
        shm.close()
        shm.unlink()

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


def _chunk(args):
    import oracle
    depth, start, stop = args
    _, num, den, ns = oracle.extract_fingerprint(_FR[start:stop], depth, zero_mean=False)
    return num, den, ns


def extract_fingerprint_chunked(frames: np.ndarray, depth: int, workers: int | None = None,
                                chunks: int | None = None):
    """The oracle's fingerprint of a long stack, computed by worker processes.

    The n_s = floor(m/d) SDA groups are split into `chunks` contiguous runs of
    whole groups (the m mod d remainder is dropped); each worker runs
    oracle.extract_fingerprint on its run and returns its partial fp64 sums
    (sum W*I, sum I^2 over its groups, ascending); the partials are added in run
    order and finalized with oracle.finalize.  This is the oracle's own
    composition (the MLE numerator and denominator are sums over the
    SDA frames), only the fp64 additions are regrouped (a relative change of the
    order of 1e-16, far below every tolerance).  Returns (K, num, den, n_s)."""
    import oracle
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    m = frames.shape[0]
    ns = oracle.sda_groups(m, depth)
    if ns < 0:
        raise oracle.OracleError(3, "extract_fingerprint_chunked")
    workers = workers or os.cpu_count() or 1
    chunks = min(ns, chunks or workers)
    bounds = [round(ns * k / chunks) for k in range(chunks + 1)]
    jobs = [(depth, bounds[k] * depth, bounds[k + 1] * depth) for k in range(chunks) if bounds[k + 1] > bounds[k]]
    shm = shared_memory.SharedMemory(create=True, size=frames.nbytes)
    try:
        np.ndarray(frames.shape, dtype=np.uint8, buffer=shm.buf)[:] = frames
        ctx = mp.get_context("spawn")
        with ctx.Pool(min(workers, len(jobs)), initializer=_init, initargs=(shm.name, frames.shape)) as pool:
            parts = pool.map(_chunk, jobs, chunksize=1)
    finally:
        shm.close()
        shm.unlink()
    num = np.zeros(frames.shape[1:])
    den = np.zeros(frames.shape[1:])
    for pn, pd, _ in parts:   # in run order
        num += pn
        den += pd
    assert sum(p[2] for p in parts) == ns
    return oracle.finalize(num, den), num, den, ns


# ---------------------------------------------------------------- worker pool for large parity tests
def _fp_job(args):
    import oracle
    name, shape, depth = args
    shm = shared_memory.SharedMemory(name=name)
    try:
        fr = np.ndarray(shape, dtype=np.uint8, buffer=shm.buf)
        K, num, den, ns = oracle.extract_fingerprint(fr, depth)
        return K, den, ns
    finally:
        shm.close()


def _res_job(args):
    import oracle
    name, shape = args
    shm = shared_memory.SharedMemory(name=name)
    try:
        q = np.ndarray(shape, dtype=np.uint8, buffer=shm.buf)
        return oracle.residual(q.astype(np.float32), zero_mean=True)
    finally:
        shm.close()


def _pce_job(args):
    from oracle import match
    R, T = args
    C = match.correlation_surface(R, T)
    p, peak, _ = match.pce_from_surface(C)
    top = np.sort(np.abs(C).ravel())[-2:]
    gap = float((top[1] - top[0]) / top[1])
    return p, peak, gap, (C if gap < 1e-4 else None)   # the surface only for a near-tie (R-19)


class OraclePool:
    """A pool of worker processes (one per host core) running oracle functions on
    arrays handed over through shared memory: fingerprints of many videos and
    residual / PCE evaluations for the full-size camera-ID parity test.  At most
    `max_pending` inputs are held at once (bounded host memory)."""

    def __init__(self, workers: int | None = None, max_pending: int | None = None):
        self.workers = workers or os.cpu_count() or 1
        self.max_pending = max_pending or 2 * self.workers
        self.pool = mp.get_context("spawn").Pool(self.workers)
        self.pending = []   # (async result, shm)

    def _share(self, a: np.ndarray):
        a = np.ascontiguousarray(a)
        shm = shared_memory.SharedMemory(create=True, size=max(1, a.nbytes))
        np.ndarray(a.shape, dtype=a.dtype, buffer=shm.buf)[:] = a
        return shm

    def _throttle(self):
        while len([p for p in self.pending if not p[0].ready()]) >= self.max_pending:
            self.pending[0][0].wait(0.05)
            self._reap()

    def _reap(self):
        for p in self.pending:
            if p[0].ready() and p[1] is not None:
                p[1].close()
                p[1].unlink()
                p[1] = None

    def fingerprint(self, frames: np.ndarray, depth: int):
        """oracle.extract_fingerprint(frames, depth) -> async (K, den, n_s)."""
        self._throttle()
        shm = self._share(frames)
        r = self.pool.apply_async(_fp_job, ((shm.name, frames.shape, depth),))
        self.pending.append([r, shm])
        return r

    def residual(self, frame: np.ndarray):
        """oracle.residual(frame, zero_mean=True) of a u8 frame -> async fp64 plane."""
        self._throttle()
        shm = self._share(frame)
        r = self.pool.apply_async(_res_job, ((shm.name, frame.shape),))
        self.pending.append([r, shm])
        return r

    def pce(self, R: np.ndarray, T: np.ndarray):
        """oracle PCE of (R, T) -> async (pce, peak, top-2 relative gap, surface)."""
        return self.pool.apply_async(_pce_job, ((R, T),))

    def close(self):
        for p in self.pending:
            p[0].wait()
        self._reap()
        self.pool.close()
        self.pool.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

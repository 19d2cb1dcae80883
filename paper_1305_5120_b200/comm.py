"""Communicators for the column-sharded solver.

The sharded phases (distributed.py) need four operations: rank/world, a flat
all-gather of equal-size shards, a broadcast and a barrier. Two ways to have
several GPUs take part:

* :class:`TorchComm` -- one process per GPU under torch.distributed (NCCL over
  NVLink on B200; gloo on CPU in the tests). Used when a caller passes a
  ``torch.distributed`` process group (``group=``), e.g. under torchrun.
* :class:`ThreadComm` -- one host thread per GPU inside ONE process, so an
  unmodified drop-in caller of ``chfsi_solve(H, Y0, config)`` (reference
  core.py:385) gets every GPU with ``devices=N``; the reference likewise takes
  its parallelism in-process (linalg.py:49-64 ``set_workers``). Backend
  ``"nccl"``: an NCCL clique over distinct GPUs (``chfsi_comm_init_all`` in
  libchfsi_b200.so, csrc/comm.cu). Backend ``"local"``: host-synchronised
  copies through shared slots -- for ranks that share one GPU (tests) or CPU
  tensors; never a performance path.

:func:`run_on_devices` starts the threads, gives each its own engine handle
and stream, and returns every rank's result (re-raising the first failure).
"""

import copy
import ctypes
import os
import threading

import numpy as np
import torch

from .errors import ChfsiError


class Comm:
    """Interface of the collectives the sharded solver uses."""

    rank = 0
    world = 1
    backend = "none"

    def all_gather_into_tensor(self, out, inp):
        raise NotImplementedError

    def broadcast(self, t, src=0):
        raise NotImplementedError

    def barrier(self):
        raise NotImplementedError

    def host_staging(self, t):
        """True when a device tensor must be staged through the host (gloo)."""
        return False


class TorchComm(Comm):
    """torch.distributed process group (``None``: the default group)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group))

    def all_gather_into_tensor(self, out, inp):
        if self.host_staging(inp):
            recv = torch.empty(out.shape, dtype=out.dtype)
            self.dist.all_gather_into_tensor(recv, inp.cpu(), group=self.group)
            out.copy_(recv)
        else:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
        return out

    def broadcast(self, t, src=0):
        if self.host_staging(t):
            h = t.cpu()
            self.dist.broadcast(h, src=src, group=self.group)
            t.copy_(h)
        else:
            self.dist.broadcast(t, src=src, group=self.group)
        return t

    def barrier(self):
        self.dist.barrier(group=self.group)

    def host_staging(self, t):
        return t.is_cuda and self.backend == "gloo"


def as_comm(group):
    """Comm for ``group``: a Comm passes through, a torch.distributed group is wrapped,
    None means the default torch.distributed group when one is initialised (else None)."""
    if group is None:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return TorchComm(None)
        return None
    if isinstance(group, Comm):
        return group
    return TorchComm(group)


def world_of(group):
    """(rank, world) of ``group``; (0, 1) without one."""
    c = as_comm(group)
    return (0, 1) if c is None else (c.rank, c.world)


class _Clique:
    """State shared by the ThreadComm ranks of one in-process group."""

    def __init__(self, devices, backend):
        self.devices = list(devices)
        self.world = len(self.devices)
        self.backend = backend
        self.barrier = threading.Barrier(self.world)
        self.slots = [None] * self.world
        self.handles = []
        self.broken = False
        if backend == "nccl":
            from . import _native
            lib = _native.load()
            devs = (ctypes.c_int * self.world)(*self.devices)
            hs = (ctypes.c_void_p * self.world)()
            _native.check("chfsi_comm_init_all", lib.chfsi_comm_init_all(self.world, devs, hs))
            self.handles = [ctypes.c_void_p(h) for h in hs]

    def abort(self):
        self.broken = True
        self.barrier.abort()
        if self.handles:
            from . import _native
            for h in self.handles:
                _native.load().chfsi_comm_abort(h)

    def close(self):
        if self.handles:
            from . import _native
            for h in self.handles:
                _native.load().chfsi_comm_destroy(h)
            self.handles = []


class ThreadComm(Comm):
    """Rank ``rank`` of an in-process clique (one host thread per rank)."""

    def __init__(self, clique, rank):
        self.clique = clique
        self.rank = rank
        self.world = clique.world
        self.backend = clique.backend

    def _wait(self):
        try:
            self.clique.barrier.wait()
        except threading.BrokenBarrierError:
            raise ChfsiError("in-process group aborted: another rank failed") from None

    def _stream(self, t):
        return torch.cuda.current_stream(t.device).cuda_stream if t.is_cuda else 0

    def all_gather_into_tensor(self, out, inp):
        if self.backend == "nccl":
            from . import _native
            nbytes = inp.numel() * inp.element_size()
            if out.numel() * out.element_size() != nbytes * self.world:
                raise ValueError("all_gather: output must hold world x input bytes")
            _native.call("chfsi_comm_allgather", self.clique.handles[self.rank],
                         ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                         nbytes, ctypes.c_void_p(self._stream(inp)))
            return out
        # local: publish the (ready) input, copy every rank's input, then wait until
        # every rank has copied before anyone may overwrite its input
        if inp.is_cuda:
            torch.cuda.current_stream(inp.device).synchronize()
        self.clique.slots[self.rank] = inp
        self._wait()
        flat = out.view(self.world, *inp.shape)
        for r in range(self.world):
            flat[r].copy_(self.clique.slots[r])
        if out.is_cuda:
            torch.cuda.current_stream(out.device).synchronize()
        self._wait()
        return out

    def broadcast(self, t, src=0):
        if self.backend == "nccl":
            from . import _native
            _native.call("chfsi_comm_broadcast", self.clique.handles[self.rank],
                         ctypes.c_void_p(t.data_ptr()), t.numel() * t.element_size(), int(src),
                         ctypes.c_void_p(self._stream(t)))
            return t
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        if self.rank == src:
            self.clique.slots[src] = t
        self._wait()
        if self.rank != src:
            t.copy_(self.clique.slots[src])
            if t.is_cuda:
                torch.cuda.current_stream(t.device).synchronize()
        self._wait()
        return t

    def barrier(self):
        self._wait()


_default_devices = None
_tls = threading.local()


def set_devices(devices):
    """Default GPU set of the drop-in entry points when a call passes neither ``group=``
    nor ``devices=`` (None or 1: one GPU). The GPU counterpart of the reference's
    in-process worker knob (linalg.py:49-64 ``set_workers`` / ``CHFSI_WORKERS``); the
    environment variable ``CHFSI_DEVICES`` (an int or a comma list) sets it too, so an
    unmodified caller of ``chfsi_solve(H, None, config)`` runs on every listed GPU."""
    global _default_devices
    _default_devices = None if devices is None else normalize_devices(devices)


def get_devices():
    if _default_devices is not None:
        return list(_default_devices)
    env = os.environ.get("CHFSI_DEVICES", "").strip()
    if not env:
        return None
    return normalize_devices(int(env) if env.isdigit() else [int(x) for x in env.split(",")])


def default_devices():
    """The default multi-GPU set for a drop-in call, or None (one GPU). Never inside a
    rank thread of an in-process group (those calls carry their own ``group``)."""
    if getattr(_tls, "inside", False):
        return None
    d = get_devices()
    return d if d is not None and len(d) > 1 else None


class inside_group:
    """Context: calls made here do not pick up the default devices again."""

    def __enter__(self):
        self.prev = getattr(_tls, "inside", False)
        _tls.inside = True

    def __exit__(self, *exc):
        _tls.inside = self.prev


def normalize_devices(devices):
    """``devices``: an int N (GPUs 0..N-1) or a sequence of CUDA ordinals."""
    if isinstance(devices, int):
        if devices < 1:
            raise ValueError("devices must be >= 1")
        return list(range(devices))
    out = [int(torch.device(d).index if not isinstance(d, int) else d) for d in devices]
    if not out:
        raise ValueError("empty device list")
    return out


def choose_backend(devices):
    """NCCL for distinct GPUs; the host-synchronised local copies when ranks share one."""
    return "nccl" if len(set(devices)) == len(devices) else "local"


def run_on_devices(devices, fn, backend=None):
    """Run ``fn(comm)`` on one host thread per entry of ``devices`` (each thread's current
    CUDA device set, with its own stream and engine handle) and return the results in
    rank order. The first exception is re-raised after every thread has ended; a
    failing rank aborts the clique so the others do not wait forever."""
    devices = normalize_devices(devices)
    if backend is None:
        backend = choose_backend(devices)
    if backend == "nccl" and len(set(devices)) != len(devices):
        raise ValueError("the nccl backend needs distinct devices")
    # the caller's pending work (e.g. the device-resident inputs the ranks copy from)
    # completes before any rank thread runs on its own stream
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    with _clique_lock:  # one in-process group at a time owns a clique
        return _run(devices, backend, fn)


# NCCL cliques are kept for the next call on the same devices (ncclCommInitAll costs
# far more than a small solve); release_devices() destroys them.
_cliques = {}
_clique_lock = threading.RLock()


def release_devices():
    """Destroy the cached in-process NCCL cliques."""
    with _clique_lock:
        for c in _cliques.values():
            c.close()
        _cliques.clear()


def _run(devices, backend, fn):
    from . import device as dev
    key = (tuple(devices), backend)
    clique = _cliques.get(key)
    if clique is None or clique.broken:
        if clique is not None:
            clique.close()
        clique = _Clique(devices, backend)
        _cliques[key] = clique
    results = [None] * clique.world
    errors = [None] * clique.world

    def body(rank):
        d = devices[rank]
        _tls.inside = True
        try:
            torch.cuda.set_device(d)
            dev.set_engine_tag(rank)
            stream = torch.cuda.Stream(device=d)
            with torch.cuda.stream(stream):
                results[rank] = fn(ThreadComm(clique, rank))
                stream.synchronize()
        except BaseException as exc:  # noqa: BLE001 - re-raised in the caller
            errors[rank] = exc
            clique.abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"chfsi-rank{r}")
               for r in range(clique.world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    clique.slots = [None] * clique.world  # drop the last call's tensors
    if clique.broken:  # an aborted clique is not reused
        clique.close()
        _cliques.pop(key, None)
    # the root cause, not a secondary "group aborted" of a waiting rank
    first = next((e for e in errors if e is not None and not _is_abort(e)), None)
    if first is None:
        first = next((e for e in errors if e is not None), None)
    if first is not None:
        raise first
    return results


def _is_abort(exc):
    return isinstance(exc, ChfsiError) and "in-process group aborted" in str(exc)


def clone_rng(seed):
    """Per-rank copy of the caller's seed / Generator: every rank must draw the same
    stream (the start block and rank-collapse columns are replicated)."""
    if isinstance(seed, np.random.Generator):
        return copy.deepcopy(seed)
    return seed

"""Rank context: one process per GPU over torch.distributed.

Replaces the reference's simulated runtime (SimRuntime / RankContext,
pkg/src/blocksim/runtime/core.py:56-121,124-218) for the calls the LBM path
makes: `rank`, `n_ranks`, `all_gather`, `all_reduce`, `barrier`.  The
per-step halo traffic does not go through this object's Python API: the
boundary-plane kernel stores the crossing directions into the neighbour's
ghost plane (peer stores over NVLink, halo.PeerHalo), with NCCL send/recv of
the contiguous runs as the fallback (halo.py).
"""
from __future__ import annotations

import os
import pickle
import socket

import torch
import torch.distributed as dist

from .errors import ValidationError


class Context:
    """Per-rank handle.  Single process when torch.distributed is not
    initialised (n_ranks == 1)."""

    def __init__(self, device=None):
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank()
            self.n_ranks = dist.get_world_size()
            self.backend = dist.get_backend()
        else:
            self.rank, self.n_ranks, self.backend = 0, 1, None
        if device is None:
            if torch.cuda.is_available():
                local = int(os.environ.get("LOCAL_RANK", self.rank))
                device = torch.device("cuda", local % max(1, torch.cuda.device_count()))
            else:
                device = torch.device("cpu")
        self.device = torch.device(device)
        self.step = 0

    @property
    def distributed(self) -> bool:
        return self.n_ranks > 1

    def all_gather(self, obj) -> dict:
        """{rank: obj} from every rank (RankContext.all_gather, core.py:95-100)."""
        if self.n_ranks == 1:
            return {0: pickle.loads(pickle.dumps(obj))}
        out = [None] * self.n_ranks
        dist.all_gather_object(out, obj)
        return {r: out[r] for r in range(self.n_ranks)}

    def all_reduce(self, values, op: str = "sum"):
        """Element-wise reduction folded in ascending rank order (core.py:82-93)."""
        scalar = isinstance(values, (int, float))
        vec = [float(values)] if scalar else [float(v) for v in values]
        gathered = self.all_gather(vec)
        acc = list(gathered[0])
        for r in range(1, self.n_ranks):
            for k, v in enumerate(gathered[r]):
                if op == "sum":
                    acc[k] = acc[k] + v
                elif op == "max":
                    acc[k] = max(acc[k], v)
                elif op == "min":
                    acc[k] = min(acc[k], v)
                else:
                    raise ValidationError(f"unknown reduction {op!r}")
        return acc[0] if scalar else acc

    def barrier(self) -> None:
        if self.n_ranks > 1:
            dist.barrier()

    def advance_step(self) -> int:
        self.step += 1
        return self.step


def init_distributed(backend: str | None = None) -> Context:
    """Initialise torch.distributed from the torchrun environment (RANK,
    WORLD_SIZE, MASTER_ADDR, MASTER_PORT) and return the rank context."""
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1 and not dist.is_initialized():
        # LBM_B200_BACKEND=gloo: several ranks sharing one GPU (host-staged
        # halos; the multi-rank bench smoke on a single-GPU box)
        backend = backend or os.environ.get("LBM_B200_BACKEND")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        import datetime
        kw = {}
        if backend == "nccl":
            dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
            torch.cuda.set_device(dev)
            kw["device_id"] = dev     # eager communicator init, device-bound barriers
        # fail instead of hanging forever if a peer dies mid-exchange
        dist.init_process_group(backend=backend, timeout=datetime.timedelta(seconds=600), **kw)
    return Context()


# ------------------------------------------------- local multi-process runs
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, n_ranks, port, backend, device, program, args, queue):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                       "RANK": str(rank), "WORLD_SIZE": str(n_ranks), "LOCAL_RANK": str(rank)})
    try:
        dist.init_process_group(backend=backend, rank=rank, world_size=n_ranks)
        if device is None:
            device = "cpu" if backend == "gloo" else None
        if device == "cuda":
            device = torch.device("cuda", rank % torch.cuda.device_count())
            torch.cuda.set_device(device)
        ctx = Context(device=device)
        res = program(ctx, *args)
        queue.put((rank, "ok", res))
    except BaseException as exc:  # report, do not hang the parent
        import traceback
        queue.put((rank, "error", f"{type(exc).__name__}: {exc}\n{traceback.format_exc()}"))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


class _ThreadGroup:
    """Shared state of the ranks of one `run(..., backend="threads")`."""

    def __init__(self, n_ranks: int):
        import threading
        self.n_ranks = n_ranks
        self.slots = [None] * n_ranks
        self.sync = threading.Barrier(n_ranks)
        self.shared = {}           # rank-visible registry (the fused halo's peer table)


class ThreadContext(Context):
    """Rank context of one thread of an in-process rank group.

    The ranks of a group are threads of one process sharing the GPU(s) it
    sees; collectives go through a barrier and a slot per rank, in rank
    order like the process transport.  On the device each rank keeps its own
    streams, so the fused peer-store halo (halo.PeerHalo) runs its real
    device-side phase protocol between the ranks' streams - without
    processes time-sliced on one GPU, and with no kernel waiting on
    another.  This is how the multi-rank device path is exercised on a
    single-GPU box; production runs use one process per GPU."""

    def __init__(self, group: _ThreadGroup, rank: int, device=None):
        self.group = group
        self.rank, self.n_ranks, self.backend = rank, group.n_ranks, "threads"
        if device is None or device == "cuda":
            device = torch.device("cuda", rank % max(1, torch.cuda.device_count())) \
                if torch.cuda.is_available() else torch.device("cpu")
        self.device = torch.device(device)
        self.step = 0

    def all_gather(self, obj) -> dict:
        g = self.group
        g.slots[self.rank] = pickle.dumps(obj)
        g.sync.wait()
        out = {r: pickle.loads(g.slots[r]) for r in range(self.n_ranks)}
        g.sync.wait()
        return out

    def barrier(self) -> None:
        self.group.sync.wait()


def _run_threads(n_ranks, program, args, device, timeout):
    import threading
    group = _ThreadGroup(n_ranks)
    results, errors = {}, []

    def body(rank):
        try:
            ctx = ThreadContext(group, rank, device)
            if ctx.device.type == "cuda":
                # each rank its own (non-blocking) main stream, as a process
                # would have: ranks must not serialise on the legacy stream
                torch.cuda.set_device(ctx.device)
                with torch.cuda.stream(torch.cuda.Stream(ctx.device)):
                    results[rank] = program(ctx, *args)
                    torch.cuda.current_stream(ctx.device).synchronize()
            else:
                results[rank] = program(ctx, *args)
        except BaseException as exc:  # report, and release ranks blocked in a collective
            import traceback
            errors.append(f"rank {rank}: {type(exc).__name__}: {exc}\n{traceback.format_exc()}")
            group.sync.abort()

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(n_ranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
        if t.is_alive():
            raise RuntimeError(f"thread rank group did not finish within {timeout} s")
    if errors:
        raise RuntimeError("rank failed:\n" + "\n".join(errors))
    return [results[r] for r in range(n_ranks)]


def run(n_ranks: int, program, *args, backend: str = "gloo", device=None,
        timeout: float = 600.0):
    """Run `program(ctx, *args)` on `n_ranks` local processes (SimRuntime.run's
    role in the reference tests).  Returns the per-rank results in rank order.
    backend="gloo", device="cuda" runs several ranks on the GPUs present
    (ranks may share one GPU; halos are then staged through the host, or go
    through CUDA IPC peer stores with LBM_B200_HALO=peer).
    backend="threads" runs the ranks as threads of this process
    (ThreadContext): the fused device-side halo between the ranks' streams."""
    import torch.multiprocessing as mp
    if n_ranks == 1:
        return [program(Context(device=device if device != "cuda" else None), *args)]
    if backend == "threads":
        return _run_threads(n_ranks, program, args, device, timeout)
    ctxmp = mp.get_context("spawn")
    queue = ctxmp.Queue()
    port = _free_port()
    procs = [ctxmp.Process(target=_worker,
                           args=(r, n_ranks, port, backend, device, program, args, queue))
             for r in range(n_ranks)]
    for p in procs:
        p.start()
    results, errors = {}, []
    for _ in range(n_ranks):
        rank, status, payload = queue.get(timeout=timeout)
        if status == "ok":
            results[rank] = payload
        else:
            errors.append(payload)
    for p in procs:
        p.join(timeout=60)
    if errors:
        raise RuntimeError("rank failed:\n" + "\n".join(errors))
    return [results[r] for r in range(n_ranks)]

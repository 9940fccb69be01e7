"""One process per GPU: the launcher `bench.py --gpus N` uses when it is not
already running under torchrun (and the multi-rank tests use on CPU).

It re-runs the given script under `torch.distributed.run` on this node with
the rendezvous on 127.0.0.1 (the container hostname may not resolve), N
ranks, RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* in each rank's environment —
exactly the command the driver's scaling run uses.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_argv(nproc: int, script: str, args, port: int | None = None):
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={int(nproc)}", "--master-addr=127.0.0.1",
            f"--master-port={port or free_port()}", script, *[str(a) for a in args]]


def under_torchrun() -> bool:
    return "WORLD_SIZE" in os.environ and "RANK" in os.environ


def spawn(nproc: int, script: str, args, env: dict | None = None, timeout: float | None = None,
          capture: bool = False) -> subprocess.CompletedProcess:
    """Run `script args` as `nproc` ranks; returns the finished process (its
    stdout is rank 0's JSON for bench.py)."""
    e = dict(os.environ)
    e.setdefault("OMP_NUM_THREADS", "1")
    if env:
        e.update(env)
    return subprocess.run(torchrun_argv(nproc, script, args), env=e, timeout=timeout,
                          text=True, stdout=subprocess.PIPE if capture else None,
                          stderr=subprocess.PIPE if capture else None)

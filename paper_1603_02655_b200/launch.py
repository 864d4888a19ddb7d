"""One-node multi-rank launcher (plumbing only): starts N ranks of a script
with torch.distributed.run, rendezvous on 127.0.0.1 at a free port.  Used by
`bench.py --gpus N` when no launcher set WORLD_SIZE, and by the gloo tests
(tests/test_multi_gloo.py), so both go through the same path."""
from __future__ import annotations

import os
import socket
import subprocess
import sys


def free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_local(nprocs: int, script: str, argv, capture: bool = False, env=None, timeout=None):
    """Run `script argv...` as `nprocs` ranks on this node (RANK, LOCAL_RANK,
    WORLD_SIZE, MASTER_ADDR=127.0.0.1, MASTER_PORT set by the launcher).
    Returns the exit code, or (exit code, stdout) with capture=True."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(int(nprocs)), "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(script)] + list(argv)
    e = dict(os.environ if env is None else env)
    e.pop("WORLD_SIZE", None)
    if capture:
        p = subprocess.run(cmd, stdout=subprocess.PIPE, text=True, env=e, timeout=timeout)
        return p.returncode, p.stdout
    return subprocess.call(cmd, env=e, timeout=timeout)

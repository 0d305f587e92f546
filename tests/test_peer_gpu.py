"""Peer-memory partitioned SSSP (gfb_peer_*, peer.cu) through the C ABI.

World sizes 1-3 under torchrun, all ranks on the one GPU of this box (CUDA
IPC maps each rank's slab into the others even on the same device, so the
device-initiated exchange and the cross-rank device barriers run exactly as
they would across NVLink).  tests/peer_worker.py checks distances bit-exact
against the oracle and predecessor trees on every rank; RMAT f32 / u32
(zero-weight ties exercise the repair rounds across ranks), grid and corpus
graphs, sources on the first and last rank, repeated calls.
"""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3])
def test_peer_partitioned_sssp(world):
    env = dict(os.environ, GFB_PEER_TIMEOUT_S="60", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(world), "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "peer_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env,
                       cwd=os.path.dirname(HERE))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("PEER_OK") == world, out[-4000:]


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_mg_one_process(parts):
    """gfb_mg_*: one host thread drives `parts` partitions, all on device 0
    here (concurrent streams of one context, lock-step host steps).  Same-
    device partitions need a hardware queue per stream, or a spinning
    barrier can block a peer's kernels behind it: CUDA_DEVICE_MAX_CONNECTIONS
    is raised for the child (one device per partition has no such limit)."""
    env = dict(os.environ, GFB_PEER_TIMEOUT_S="20", CUDA_DEVICE_MAX_CONNECTIONS="32")
    r = subprocess.run([sys.executable, os.path.join(HERE, "mg_worker.py"), str(parts)],
                       capture_output=True, text=True, timeout=900, env=env,
                       cwd=os.path.dirname(HERE))
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MG_OK" in out, out[-4000:]

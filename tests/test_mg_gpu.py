"""Partitioned SSSP kernels (gfb_part_*, mg.cu) on one GPU: P partitions
simulated in one process (exchange by concatenation), plus the NCCL protocol
with world_size 1.  Distances must equal the f32 / u32 oracle bit for bit."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2212_08200_b200 import mg

pytestmark = pytest.mark.gpu


def _graph(scale, wkind=1, seed=1):
    s, d, wb = O.rmat_edges(scale, 16, seed=seed, wkind=wkind)
    n = 1 << scale
    wv = wb.view(np.float32).astype(np.float64) if wkind else wb.astype(np.float64)
    ro, col, val = O.build_csr(n, s, d, wv)
    return n, ro, col, (val.astype(np.float32) if wkind else val.astype(np.uint32))


@pytest.mark.parametrize("parts", [1, 3, 4])
def test_partitioned_kernels_match_oracle(ctx, parts):
    n, ro, col, w = _graph(14)
    rs = mg.edge_balanced_ranges(ro, parts)
    engines = [mg.GfbPart(n, int(rs[p]), int(rs[p + 1]), *mg.slice_csr(ro, col, w, rs[p], rs[p + 1]),
                          ctx=ctx) for p in range(parts)]
    got, steps = mg.sssp_simulated(engines, rs, 0)
    want, _ = O.dijkstra(n, ro, col, w, 0, "f32")
    assert np.array_equal(got, want)
    # nonzero source on another partition
    src = int(rs[-2]) + 1 if parts > 1 else 5
    got, _ = mg.sssp_simulated(engines, rs, src)
    want, _ = O.dijkstra(n, ro, col, w, src, "f32")
    assert np.array_equal(got, want)


def test_partitioned_u32_matches_oracle(ctx):
    n, ro, col, w = _graph(12, wkind=0)
    rs = mg.edge_balanced_ranges(ro, 4)
    engines = [mg.GfbPart(n, int(rs[p]), int(rs[p + 1]), *mg.slice_csr(ro, col, w, rs[p], rs[p + 1]),
                          ctx=ctx) for p in range(4)]
    got, _ = mg.sssp_simulated(engines, rs, 0)
    want, _ = O.dijkstra(n, ro, col, w, 0, "u32")
    fin = want != np.iinfo(np.uint64).max
    assert np.array_equal(got[fin].astype(np.uint64), want[fin])
    assert np.all(got[~fin] == 0xFFFFFFFF)


def test_nccl_protocol_world1(ctx):
    import torch
    import torch.distributed as dist
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        n, ro, col, w = _graph(12)
        rs = mg.edge_balanced_ranges(ro, 1)
        eng = mg.GfbPart(n, 0, n, *mg.slice_csr(ro, col, w, 0, n), ctx=ctx)
        d, pred, st = mg.sssp_partitioned(eng, rs, 0, device=torch.device("cuda", 0),
                                          want_pred=True)
        want, _ = O.dijkstra(n, ro, col, w, 0, "f32")
        assert np.array_equal(d, want)
        assert O.check_pred_tree(n, ro, col, w, d, 0, pred) == -1
    finally:
        dist.destroy_process_group()

"""Host-side logic of the N > 1 bench path ("replicas only") on
CPU with the gloo backend, world size 2: max-over-ranks timing, whole-job
value, and the reference arm's rank != 0 early exit."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    ms = bench.max_over_ranks(100.0 + 50.0 * rank)       # rank 1 is the slow one
    val = bench.whole_job_value(ws, 4.0e12, ms)
    out[rank] = (ms, val)
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    ws, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
        res = dict(out)
    for r in range(ws):
        ms, val = res[r]
        assert ms == 150.0                                   # the max, on every rank
        assert val == pytest.approx(2 * 4.0e12 / 0.150 / 1e9)


def test_single_process_unchanged():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(12.5) == 12.5
    assert bench.whole_job_value(1, 1e9, 1000.0) == pytest.approx(1.0)


def test_reference_arm_nonzero_rank_exits_without_work(monkeypatch, capsys):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    args = type("A", (), {"steps": 1, "warmup": 0})()
    assert bench.run_reference(args, bench.CONFIGS[1]) == 0
    assert capsys.readouterr().out == ""

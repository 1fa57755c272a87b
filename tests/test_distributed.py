"""Multi-process sharding logic (CPU, gloo, world_size 2).

The shard split and the count all-reduce are the same code the GPU path uses
(paper_2604_01059_b200.distributed); on CPU the per-rank counts come from the
C oracle instead of the device.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden_path
from oracle import coracle
from paper_2604_01059_b200.distributed import count_outputs_sharded, gpu_counter, shard_range


@pytest.mark.parametrize("total", [0, 1, 63, 64, 65, 1000, 4096, 123457])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(total, world):
    spans = [shard_range(total, r, world) for r in range(world)]
    pos = 0
    for first, count in spans:
        assert first == pos or count == 0
        assert first % 64 == 0 or count == 0
        pos = first + count if count else pos
    assert sum(c for _, c in spans) == total


def _oracle_counter(path):
    model = coracle.OracleModel.load(path)

    def run(seed, first, shots):
        cols = model.sample(shots, seed, first)
        return torch.from_numpy(np.unpackbits(cols.view(np.uint8), axis=1).sum(axis=1).astype(np.int64))
    return run, model.num_outputs


def _worker(rank, world, port, path, total, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        counter, nout = _oracle_counter(path)
        counts = count_outputs_sharded(total, seed, nout, counter)
        if rank == 0:
            np.save(out, counts)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,total", [("c2_surface_d3_xmem_t", 20000), ("c4_color_d5_rz3", 3001)])
def test_sharded_counts_equal_single_process(name, total, tmp_path):
    path = golden_path(name)
    out = str(tmp_path / "counts.npy")
    mp.start_processes(_worker, args=(2, _free_port(), path, total, 7, out), nprocs=2, join=True,
                       start_method="spawn")
    counter, _ = _oracle_counter(path)
    single = counter(7, 0, total).numpy().astype(np.uint64)
    assert np.array_equal(np.load(out), single)


class _HostSampler:
    """Stand-in for CompiledSampler with the device entry points gpu_counter
    calls (count_device / check_errors), counting with the C oracle into the
    host memory the pointer names."""

    def __init__(self, path):
        self.model = coracle.OracleModel.load(path)
        self.num_outputs = self.model.num_outputs
        self.device = 0
        self.calls = []

    def count_device(self, seed, first, shots, ptr, stream):
        import ctypes
        self.calls.append((seed, first, shots))
        cols = self.model.sample(shots, seed, first)
        add = np.unpackbits(cols.view(np.uint8), axis=1).sum(axis=1).astype(np.int64)
        buf = np.ctypeslib.as_array((ctypes.c_int64 * self.num_outputs).from_address(ptr))
        buf += add  # zxs_count_device adds to the caller's counts

    def check_errors(self, stream):
        pass


def _gpu_counter_worker(rank, world, port, path, total, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cs = _HostSampler(path)
        counts = count_outputs_sharded(total, seed, cs.num_outputs, gpu_counter(cs, stream=0, device="cpu"))
        np.save(out + f".{rank}.npy", counts)
        np.save(out + f".calls{rank}.npy", np.array(cs.calls, dtype=np.int64).reshape(-1, 3))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,total", [("c2_surface_d3_xmem_t", 10000), ("steane_inject", 4097)])
def test_gpu_counter_path_world2(name, total, tmp_path):
    """The sampler-backed counter (gpu_counter -> count_device) under a 2-rank
    gloo group: each rank counts its own 64-aligned shot range once, and both
    ranks end with the single-process counts."""
    path = golden_path(name)
    out = str(tmp_path / "c")
    mp.start_processes(_gpu_counter_worker, args=(2, _free_port(), path, total, 5, out), nprocs=2, join=True,
                       start_method="spawn")
    counter, _ = _oracle_counter(path)
    single = counter(5, 0, total).numpy().astype(np.uint64)
    spans = [tuple(np.load(out + f".calls{r}.npy").ravel()) for r in range(2)]
    assert spans == [(5,) + shard_range(total, r, 2) for r in range(2)]
    for r in range(2):
        assert np.array_equal(np.load(out + f".{r}.npy"), single)

"""Multi-GPU hashing (SURVEY 8(e) "Hashing"): LPT placement, the exact-size digest gather
(ranks as threads and as gloo processes, world_size 2, on CPU with stand-in digests), and on
the GPU: per-rank hashing + gather against the C oracle, and the one-process multi-device
host path (b2l_init over the same B200 twice)."""
import heapq
import os

import numpy as np
import pytest

from paper_2601_12713_b200 import multigpu, sharded


def lpt_oracle(lens, parts):
    """Textbook LPT: longest first (stable), each to the least-loaded part (lowest index on ties)."""
    owner = [0] * len(lens)
    heap = [(0, p) for p in range(parts)]
    for i in sorted(range(len(lens)), key=lambda i: -int(lens[i])):
        ld, p = heapq.heappop(heap)
        owner[i] = p
        heapq.heappush(heap, (ld + int(lens[i]), p))
    return owner


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_lpt_partition_matches_textbook_lpt(parts):
    rng = np.random.default_rng(parts)
    for n in (0, 1, 5, 1000):
        lens = np.exp(rng.uniform(np.log(1024), np.log(1 << 20), n)).astype(np.uint64)
        lens[: n // 4] = 40_000  # equal sizes among them: dealt in index order
        owner, load = multigpu.lpt_partition(lens, parts)
        assert owner.tolist() == lpt_oracle(lens, parts)
        assert [int(x) for x in load] == [int(lens[owner == p].sum()) for p in range(parts)]
        if n:
            assert int(load.max()) - int(load.min()) <= int(lens.max())


def test_lpt_equal_sizes_round_robin():
    owner, load = multigpu.lpt_partition(np.full(10, 7, np.uint64), 4)
    assert owner.tolist() == [0, 1, 2, 3, 0, 1, 2, 3, 0, 1] and load.tolist() == [21, 21, 14, 14]


def _gather_case(comm, n=257, parts=None):
    """Stand-in digests f(i) for the buffers LPT places on this rank -> rank 0 must see f in
    global order."""
    import torch
    parts = parts or comm.size
    lens = (np.arange(n, dtype=np.uint64) * 7919 % 1000) + 1
    owner, _ = multigpu.lpt_partition(lens, parts)
    mine = np.nonzero(owner == comm.rank)[0]
    dig = torch.from_numpy((mine.astype(np.int64) * 1000003) ^ 0x5A5A)
    return multigpu.gather_digests(dig, torch.from_numpy(mine.astype(np.int64)), n, comm)


@pytest.mark.parametrize("g", [2, 3, 4])
def test_gather_digests_local_ranks(g):
    import threading
    comms = sharded.LocalComm.group(g)
    res = [None] * g
    th = [threading.Thread(target=lambda r=r: res.__setitem__(r, _gather_case(comms[r]))) for r in range(g)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    want = (np.arange(257, dtype=np.int64) * 1000003) ^ 0x5A5A
    assert res[0].numpy().tolist() == want.tolist() and all(r is None for r in res[1:])


def _gloo_worker(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = _gather_case(sharded.TorchComm())
        if rank == 0:
            want = (np.arange(257, dtype=np.int64) * 1000003) ^ 0x5A5A
            with open(result_path, "w") as f:
                f.write("ok" if got.numpy().tolist() == want.tolist() else "mismatch")
        else:
            assert got is None
    finally:
        dist.destroy_process_group()


def test_gather_digests_gloo_world_size_2(tmp_path):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "result.txt"
    mp.spawn(_gloo_worker, args=(2, port, str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"


def _payload_slab(lens, seed, dev):
    import torch

    from oracle import hash_ref  # the checker: payload bytes and digests
    offs = np.zeros(len(lens), np.int64)
    if len(lens) > 1:
        offs[1:] = np.cumsum((np.asarray(lens, np.int64) + 16 + 255) // 256 * 256)[:-1] + np.arange(1, len(lens)) % 16
    host = np.zeros(int(offs[-1] + lens[-1]) + 16, np.uint8)
    pays = [hash_ref.payload(int(n), seed, i) for i, n in enumerate(lens)]
    for o, p in zip(offs, pays):
        host[o:o + len(p)] = np.frombuffer(p, np.uint8)
    want = [hash_ref.fold64_c(p) for p in pays]
    return torch.from_numpy(host).to(dev), offs, want, host


@pytest.mark.gpu
@pytest.mark.parametrize("g", [2, 4])
def test_hash_sharded_local_ranks_vs_oracle(cuda, g):
    """A ragged global batch placed by LPT over g ranks (threads sharing the B200): every rank
    hashes its resident buffers, rank 0 gets all digests in global order."""
    import threading

    import torch
    rng = np.random.default_rng(g)
    lens = np.exp(rng.uniform(np.log(1), np.log(300_000), 600)).astype(np.int64)
    slab, offs, want, _ = _payload_slab(lens, 5, cuda)
    owner, _ = multigpu.lpt_partition(lens.astype(np.uint64), g)
    comms = sharded.LocalComm.group(g)
    res = [None] * g

    def rank(r):
        torch.cuda.set_device(cuda)
        mine = np.nonzero(owner == r)[0]
        ptrs = torch.from_numpy(offs[mine]).to(cuda) + slab.data_ptr()
        ln = torch.from_numpy(lens[mine]).to(cuda)
        s = torch.cuda.Stream(cuda)
        with torch.cuda.stream(s):
            res[r] = multigpu.hash_sharded(ptrs, ln, torch.from_numpy(mine.astype(np.int64)).to(cuda), len(lens),
                                           comms[r], stream=s)
        s.synchronize()
    th = [threading.Thread(target=rank, args=(r,)) for r in range(g)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    got = [int(x) & (2**64 - 1) for x in res[0].cpu().numpy().view(np.uint64)]
    assert got == want


@pytest.mark.gpu
def test_hash_host_multi_vs_oracle(cuda):
    from paper_2601_12713_b200 import EmptyPayload
    rng = np.random.default_rng(9)
    lens = np.exp(rng.uniform(np.log(1), np.log(1 << 20), 3000)).astype(np.int64)
    lens[17] = (33 << 20) + 5  # a K2-sized buffer inside one device's range
    _, offs, want, host = _payload_slab(lens, 8, "cpu")
    ptrs = (offs.astype(np.uint64) + np.uint64(host.ctypes.data))
    multigpu.init([0, 0, 0])  # three "devices" on the one B200: three ranges, three host threads
    try:
        assert multigpu.devices() == [0, 0, 0]
        out = np.zeros(len(lens), np.uint64)
        multigpu.hash_host_arrays_multi(ptrs, lens.astype(np.uint64), out)
        assert [int(x) for x in out] == want
        pays = [bytes(host[o:o + n]) for o, n in zip(offs[:50], lens[:50])]
        assert multigpu.hash_batch_multi(pays) == want[:50]
        with pytest.raises(EmptyPayload):
            multigpu.hash_batch_multi([b"x", b""])
    finally:
        multigpu.shutdown()
    assert multigpu.devices() == []

"""GPU parity of the K1 hash kernel (through the C ABI) against the oracle
and the reference-generated golden digests.  Bit-exact."""
import json
import os

import numpy as np
import pytest

from oracle import hash_ref

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hash_vectors.json")))


def _dev_buffers(cuda, payloads, align=256, offsets=None):
    """Pack payloads into one device slab; returns (slab, ptrs tensor, lens tensor)."""
    import torch
    offs, pos = [], 0
    for i, p in enumerate(payloads):
        o = offsets[i] if offsets is not None else 0
        pos = (pos + align - 1) // align * align + o
        offs.append(pos)
        pos += len(p)
    host = np.zeros(pos + 64, dtype=np.uint8)
    for o, p in zip(offs, payloads):
        host[o:o + len(p)] = np.frombuffer(p, dtype=np.uint8)
    slab = torch.from_numpy(host).to(cuda)
    base = slab.data_ptr()
    ptrs = torch.tensor([base + o for o in offs], dtype=torch.int64, device=cuda)
    lens = torch.tensor([len(p) for p in payloads], dtype=torch.int64, device=cuda)
    return slab, ptrs, lens


def _device_digests(cuda, payloads, offsets=None, order=None):
    import torch
    from paper_2601_12713_b200 import hash_device
    from paper_2601_12713_b200.hashing import to_u64_list
    slab, ptrs, lens = _dev_buffers(cuda, payloads, offsets=offsets)
    out = torch.full((len(payloads),), -1, dtype=torch.int64, device=cuda)
    ord_t = None if order is None else torch.tensor(order, dtype=torch.int32, device=cuda)
    hash_device(ptrs, lens, out, order=ord_t)
    torch.cuda.synchronize()
    return to_u64_list(out)


def test_ts_vectors_hash_bytes(cuda):
    from paper_2601_12713_b200 import hash_bytes
    for hexp, want in GOLD["ts_vectors"]:
        assert hash_bytes(bytes.fromhex(hexp)) == int(want), hexp


def test_stability_vector(cuda):
    from paper_2601_12713_b200 import hash_bytes
    assert hash_bytes(bytes(range(256)) * 4096) == int(GOLD["stability"]["digest"])


def test_every_length_1_to_4096_device_and_host(cuda):
    from paper_2601_12713_b200 import hash_batch
    bl = GOLD["by_length"]
    payloads = [hash_ref.payload(n, bl["seed"], n) for n in range(1, 4097)]
    want = [int(d) for d in bl["digests"]]
    assert _device_digests(cuda, payloads) == want
    assert hash_batch(payloads) == want


def _variants():
    import ctypes
    from paper_2601_12713_b200 import _lib
    n = ctypes.c_int(0)
    _lib.check(_lib.lib().b2l_hash_select_variant(-1, ctypes.byref(n)))
    return list(range(n.value))


@pytest.fixture(params=range(16))
def variant(request, cuda):
    from paper_2601_12713_b200 import _lib
    if request.param >= len(_variants()):
        pytest.skip("no such variant")
    _lib.check(_lib.lib().b2l_hash_select_variant(request.param, None))
    yield request.param
    _lib.check(_lib.lib().b2l_hash_select_variant(-2, None))


def test_all_variants_misaligned_ragged(variant):
    import torch
    cuda = torch.device("cuda:0")
    rng = np.random.default_rng(10 + variant)
    lens = [int(x) for x in rng.integers(1, 5000, size=200)] + [1, 7, 8, 9, 15, 16, 17, 127, 128, 129, 383, 384,
                                                                  385, 511, 512, 513, 1023, 1024, 1025, 2047]
    offs = [int(x) for x in rng.integers(0, 16, size=len(lens))]
    payloads = [hash_ref.payload(n, 21, i) for i, n in enumerate(lens)]
    want = [hash_ref.fold64_c(p) for p in payloads]
    assert _device_digests(cuda, payloads, offsets=offs) == want
    order = list(np.argsort(-np.array(lens), kind="stable"))
    assert _device_digests(cuda, payloads, offsets=offs, order=order) == want
    z = _device_digests(cuda, [b"ab", b"", b"c" * 1000, b""])
    assert z[1] == 0 and z[3] == 0 and z[0] == hash_ref.fold64_c(b"ab")


def test_misaligned_starts_0_to_15(cuda):
    rng = np.random.default_rng(1)
    for off in range(16):
        lens = [int(x) for x in rng.integers(1, 3000, size=40)] + [1, 7, 8, 9, 15, 16, 17, 255, 256, 257]
        payloads = [hash_ref.payload(n, 99, 7 * n + off) for n in lens]
        got = _device_digests(cuda, payloads, offsets=[off] * len(payloads))
        assert got == [hash_ref.fold64_c(p) for p in payloads], off


def test_mixed_alignment_in_one_warp(cuda):
    rng = np.random.default_rng(2)
    lens = [int(x) for x in rng.integers(1, 20000, size=300)]
    offs = [int(x) for x in rng.integers(0, 16, size=300)]
    payloads = [hash_ref.payload(n, 5, i) for i, n in enumerate(lens)]
    assert _device_digests(cuda, payloads, offsets=offs) == [hash_ref.fold64_c(p) for p in payloads]


def test_large_golden_payloads(cuda):
    payloads = [hash_ref.payload(it["len"], it["seed"], it["content_id"]) for it in GOLD["large"]]
    want = [int(it["digest"]) for it in GOLD["large"]]
    assert _device_digests(cuda, payloads) == want


def test_ragged_longest_first_order(cuda):
    rng = np.random.default_rng(3)
    lens = [int(np.exp(x)) for x in rng.uniform(np.log(1024), np.log(1 << 20), size=64)]
    payloads = [hash_ref.payload(n, 17, i) for i, n in enumerate(lens)]
    order = list(np.argsort(-np.array(lens), kind="stable"))
    want = [hash_ref.fold64_c(p) for p in payloads]
    assert _device_digests(cuda, payloads, order=order) == want
    assert _device_digests(cuda, payloads) == want


def test_split_pairs_chunk_edges_and_reuse(cuda):
    """Ragged batches fold their longest buffers with warp pairs (lo / hi 32-bit chains,
    b2l_hash.cu "split pair"): lengths at the 64 KiB eligibility edge and around the 4 KiB
    chunks (tails of 1..7 bytes, a last chunk with no full word), unaligned long buffers (warp A
    alone), zero-length entries, and more long buffers than pairs so every pair folds several
    (its ring slots and barrier phases carry over)."""
    rng = np.random.default_rng(31)
    edge = [64 << 10, (64 << 10) - 1, (64 << 10) + 1, (64 << 10) + 7, 4096 * 17, 4096 * 17 + 1, 4096 * 17 + 8,
            4096 * 17 + 9, 4096 * 33 - 1, 4096 * 40 + 3, (1 << 20) + 5, 1 << 20, 0, 0]
    lens = edge + [int(x) for x in rng.integers(64 << 10, 300 << 10, size=420)] + \
        [int(x) for x in rng.integers(1, 5000, size=200)]
    offs = [0] * len(lens)
    for i in range(0, len(lens), 7):
        offs[i] = int(rng.integers(1, 16))  # unaligned: not split-eligible
    payloads = [hash_ref.payload(n, 23, i) for i, n in enumerate(lens)]
    want = [hash_ref.fold64_c(p) if p else 0 for p in payloads]
    order = list(np.argsort(-np.array(lens), kind="stable"))
    assert _device_digests(cuda, payloads, offsets=offs, order=order) == want
    assert _device_digests(cuda, payloads, order=order) == want


def test_host_batch_merged_copy_runs(cuda):
    """b2l_hash_host merges buffers that follow each other in host memory -- adjacent, or with a
    gap inside pages the two buffers touch -- into one DMA (b2l_api.cu copy plan): gaps of
    0..4096 bytes at every alignment, buffers out of address order, a buffer inside another's
    run, and buffers in separate allocations, pinned and pageable."""
    import torch
    from paper_2601_12713_b200.hashing import hash_host_arrays
    rng = np.random.default_rng(41)
    lens = [int(x) for x in rng.integers(1, 20000, size=600)]
    gaps = [int(rng.choice([0, 0, 1, 7, 15, 16, 100, 255, 4000, 4096, 4097, 9000])) for _ in lens]
    total = sum(lens) + sum(gaps) + 64
    pinned = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    host = pinned.numpy()
    host[:] = np.frombuffer(rng.bytes(total), np.uint8)
    offs, pos = [], 3
    for n, g in zip(lens, gaps):
        offs.append(pos)
        pos += n + g
    payloads = [bytes(host[o:o + n]) for o, n in zip(offs, lens)]
    base = pinned.data_ptr()
    order = np.arange(len(lens))
    order[100:200] = order[100:200][::-1]  # a stretch out of address order
    ptrs = np.array([base + offs[i] for i in order], np.uint64)
    ln = np.array([lens[i] for i in order], np.uint64)
    extra = [np.frombuffer(rng.bytes(n), np.uint8).copy() for n in (5, 4096, 70001)]  # pageable, separate
    inside = (offs[10] + 1, max(lens[10] - 1, 1))  # inside another buffer's run
    ptrs = np.concatenate([ptrs[:50], np.array([e.ctypes.data for e in extra], np.uint64), ptrs[50:],
                           np.array([base + inside[0]], np.uint64)])
    ln = np.concatenate([ln[:50], np.array([e.size for e in extra], np.uint64), ln[50:],
                         np.array([inside[1]], np.uint64)])
    want = [hash_ref.fold64_c(payloads[i]) for i in order]
    want = want[:50] + [hash_ref.fold64_c(e.tobytes()) for e in extra] + want[50:] + \
        [hash_ref.fold64_c(bytes(host[inside[0]:inside[0] + inside[1]]))]
    out = np.zeros(ptrs.size, np.uint64)
    hash_host_arrays(ptrs, ln, out)
    assert out.tolist() == want


def test_zero_length_gets_reserved_digest_and_host_raises(cuda):
    from paper_2601_12713_b200 import EmptyPayload, hash_batch, hash_bytes
    payloads = [b"abc", b"", b"x" * 100]
    got = _device_digests(cuda, [p if p else b"" for p in payloads])
    assert got[1] == 0 and got[0] == hash_ref.fold64_c(b"abc")
    with pytest.raises(EmptyPayload):
        hash_bytes(b"")
    with pytest.raises(EmptyPayload):
        hash_batch(payloads)


def test_many_uniform_buffers_generated_on_device(cuda):
    """C2-shaped slice: 20k x 40,000 B, 25% duplicates, generated by the device
    payload generator; digests checked against the C oracle on host copies."""
    import torch
    from paper_2601_12713_b200 import _lib, hash_device
    from paper_2601_12713_b200.hashing import to_u64_list
    n, size = 20000, 40000
    rng = np.random.default_rng(4)
    cids = np.arange(n, dtype=np.int64)
    dup = rng.random(n) < 0.25
    cids[dup] = rng.integers(0, n, size=int(dup.sum()))
    offs = torch.arange(n, dtype=torch.int64, device=cuda) * size
    lens = torch.full((n,), size, dtype=torch.int64, device=cuda)
    slab = torch.empty(n * size, dtype=torch.uint8, device=cuda)
    c = torch.from_numpy(cids).to(cuda)
    rc = _lib.lib().b2l_fill_payloads(slab.data_ptr(), offs.data_ptr(), lens.data_ptr(), c.data_ptr(), n, 2,
                                      torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    ptrs = offs + slab.data_ptr()
    out = torch.empty(n, dtype=torch.int64, device=cuda)
    hash_device(ptrs, lens, out)
    torch.cuda.synchronize()
    got = np.array(to_u64_list(out), dtype=np.uint64)
    host = slab.cpu().numpy()
    hp = np.array([host.ctypes.data + i * size for i in range(n)], dtype=np.uint64)
    want = hash_ref.fold64_c_batch(hp, np.full(n, size, dtype=np.uint64), threads=os.cpu_count() or 1)
    assert np.array_equal(got, want)
    # duplicates hash equal, the generator is content-addressed
    i = int(np.nonzero(dup)[0][0])
    assert got[i] == got[cids[i]] or cids[i] == i


def test_hash_tensors_api(cuda):
    import torch
    from paper_2601_12713_b200 import hash_tensors
    from paper_2601_12713_b200.hashing import to_u64_list
    ts = [torch.arange(n, dtype=torch.float32, device=cuda) for n in (1, 3, 1000, 77777)]
    got = to_u64_list(hash_tensors(ts))
    want = [hash_ref.fold64_c(t.cpu().numpy().tobytes()) for t in ts]
    assert got == want


def test_buffer_larger_than_4GiB(cuda):
    import torch
    from paper_2601_12713_b200 import _lib, hash_device
    from paper_2601_12713_b200.hashing import to_u64_list
    size = (1 << 32) + 12345
    slab = torch.empty(size + 16, dtype=torch.uint8, device=cuda)
    z = torch.zeros(1, dtype=torch.int64, device=cuda)
    ln = torch.tensor([size], dtype=torch.int64, device=cuda)
    cid = torch.tensor([77], dtype=torch.int64, device=cuda)
    _lib.check(_lib.lib().b2l_fill_payloads(slab.data_ptr(), z.data_ptr(), ln.data_ptr(), cid.data_ptr(), 1, 9,
                                            torch.cuda.current_stream().cuda_stream))
    out = torch.empty(1, dtype=torch.int64, device=cuda)
    hash_device(z + slab.data_ptr(), ln, out)
    torch.cuda.synchronize()
    host = slab[:size].cpu().numpy()
    want = hash_ref.fold64_c_batch(np.array([host.ctypes.data], dtype=np.uint64),
                                   np.array([size], dtype=np.uint64))
    assert to_u64_list(out)[0] == int(want[0])


# ----------------------------------------------------------------------------- K2 (whole-GPU fold)
def _k2_digest(cuda, slab, off, n):
    import torch
    from paper_2601_12713_b200.hashing import hash_large, to_u64_list
    out = torch.zeros(1, dtype=torch.int64, device=cuda)
    hash_large(slab.data_ptr() + off, n, out.data_ptr())
    torch.cuda.synchronize()
    return to_u64_list(out)[0]


def test_k2_small_lengths_and_offsets(cuda):
    import torch
    rng = np.random.default_rng(31)
    host = np.frombuffer(hash_ref.payload(1 << 20, 5, 1), dtype=np.uint8)
    slab = torch.from_numpy(host.copy()).to(cuda)
    cases = [(o, n) for o in range(16) for n in (1, 2, 7, 8, 9, 15, 16, 17, 63, 64, 65, 255)]
    cases += [(int(rng.integers(0, 64)), int(rng.integers(1, 200_000))) for _ in range(40)]
    cases += [(3, 32768 * 8 - 5), (0, 32768 * 8), (8, 32768 * 8 + 8), (5, (1 << 20) - 64)]
    for off, n in cases:
        assert _k2_digest(cuda, slab, off, n) == hash_ref.fold64_c(host[off:off + n].tobytes()), (off, n)


def test_k2_multi_round_buffer_and_routing(cuda):
    """256 MiB + 3 bytes (C3-sized, many rounds of the co-resident grid), misaligned."""
    import torch
    from paper_2601_12713_b200 import _lib, hash_tensors
    from paper_2601_12713_b200.hashing import to_u64_list
    size = (256 << 20) + 3
    slab = torch.empty(size + 16, dtype=torch.uint8, device=cuda)
    z = torch.zeros(1, dtype=torch.int64, device=cuda)
    ln = torch.tensor([size + 16], dtype=torch.int64, device=cuda)
    cid = torch.tensor([4242], dtype=torch.int64, device=cuda)
    _lib.check(_lib.lib().b2l_fill_payloads(slab.data_ptr(), z.data_ptr(), ln.data_ptr(), cid.data_ptr(), 1, 3,
                                            torch.cuda.current_stream().cuda_stream))
    host = slab.cpu().numpy()
    for off in (0, 5):
        want = hash_ref.fold64_c_batch(np.array([host.ctypes.data + off], dtype=np.uint64),
                                       np.array([size], dtype=np.uint64))[0]
        assert _k2_digest(cuda, slab, off, size) == int(want), off
    # hash_tensors routes >= 32 MiB buffers to K2 and the rest to the batch kernel
    ts = [slab[:size], slab[1:1001], slab[:40 << 20]]
    got = to_u64_list(hash_tensors(ts))
    want = [hash_ref.fold64_c(t.cpu().numpy().tobytes()) for t in ts]
    assert got == want


def test_k2_many_ragged_vs_oracle(cuda):
    """b2l_hash_large_many: 21 buffers (two launches of up to 16), ragged and misaligned, from
    one word to 40 MiB + 7 (full and partial chunks, one- and multi-round buffers), vs the C oracle
    and vs one b2l_hash_large per buffer."""
    import torch
    from paper_2601_12713_b200.hashing import hash_large, hash_large_many
    rng = np.random.default_rng(21)
    lens = [1, 7, 8, 4095, 49152, 49153, (40 << 20) + 7, 3 << 20] + [int(x) for x in rng.integers(1, 3 << 20, 13)]
    offs, o = [], 0
    for n in lens:
        o += int(rng.integers(0, 8))
        offs.append(o)
        o += n
    slab = torch.randint(0, 256, (o + 8,), dtype=torch.uint8, device=cuda)
    ptrs = [slab.data_ptr() + x for x in offs]
    out = torch.zeros(len(lens), dtype=torch.int64, device=cuda)
    hash_large_many(ptrs, lens, out.data_ptr())
    one = torch.zeros(len(lens), dtype=torch.int64, device=cuda)
    for i, (p, n) in enumerate(zip(ptrs, lens)):
        hash_large(p, n, one.data_ptr() + 8 * i)
    torch.cuda.synchronize()
    host = slab.cpu().numpy()
    want = hash_ref.fold64_c_batch(np.array([host.ctypes.data + x for x in offs], dtype=np.uint64),
                                   np.array(lens, dtype=np.uint64))
    assert out.cpu().numpy().view(np.uint64).tolist() == want.tolist()
    assert torch.equal(out, one)
    with pytest.raises(Exception):
        hash_large_many(ptrs[:2], [5, 0], out.data_ptr())


def test_hash_tensors_on_side_stream(cuda):
    """hash_tensors(stream=...) with K2 and K1 buffers: every torch copy/scatter of the call is
    ordered on the caller's stream (a torch Stream or a raw handle)."""
    import torch
    from paper_2601_12713_b200 import hash_tensors
    from paper_2601_12713_b200.hashing import to_u64_list
    g = torch.Generator(device=cuda).manual_seed(5)
    slab = torch.randint(0, 256, ((40 << 20) + (33 << 20) + 4096,), dtype=torch.uint8, device=cuda, generator=g)
    ts = [slab[:(40 << 20) + 1], slab[(40 << 20) + 3:(40 << 20) + 1003], slab[-(33 << 20):]]
    want = [hash_ref.fold64_c(t.cpu().numpy().tobytes()) for t in ts]
    side = torch.cuda.Stream(device=cuda)
    for st in (side, side.cuda_stream):
        got = hash_tensors(ts, stream=st)
        side.synchronize()
        assert to_u64_list(got) == want


# ----------------------------------------------------------------------------- collision audit
def test_audit_reference_cases(cuda):
    from paper_2601_12713_b200 import CollisionAuditStore, audit_observe, hash_bytes
    store = CollisionAuditStore()
    h = hash_bytes(b"abcdef")
    audit_observe(store, h, b"abcdef")
    audit_observe(store, h, b"abcdef")
    assert store.collision_count == 0 and len(store) == 1
    store = CollisionAuditStore()
    audit_observe(store, 42, b"first")
    audit_observe(store, 42, b"second")
    assert store.collision_count == 1
    audit_observe(store, 42, b"third")
    assert store.collision_count == 2
    audit_observe(store, 42, b"first")
    assert store.collision_count == 2


def test_audit_random_vs_oracle(cuda):
    from paper_2601_12713_b200.hashing import audit_payloads
    rng = np.random.default_rng(9)
    for trial in range(20):
        n = int(rng.integers(1, 400))
        pool = [hash_ref.payload(int(rng.integers(1, 3000)), 4, i) for i in range(int(rng.integers(1, 30)))]
        obs = []
        for _ in range(n):
            p = pool[int(rng.integers(0, len(pool)))]
            if rng.random() < 0.1 and len(p) > 1:  # near-miss: one flipped byte / truncated
                p = p[:-1] if rng.random() < 0.5 else bytes([p[0] ^ 1]) + p[1:]
            obs.append((int(rng.integers(0, 8)), p))
        assert audit_payloads([h for h, _ in obs], [p for _, p in obs]) == hash_ref.audit_ref(obs), trial


def test_single_buffer_routing_around_k2_solo_threshold(cuda):
    """A call hashing ONE buffer goes to K2 from 96 KiB (b2l_hash_bytes, hash_tensors) and
    small calls take the one-DMA staging path; every route equals the oracle."""
    import torch
    from paper_2601_12713_b200 import hash_batch, hash_bytes, hash_tensors
    from paper_2601_12713_b200.hashing import to_u64_list
    base = hash_ref.payload(1 << 20, 9, 2)
    for n in (1, 15, 4096, 65536, (96 << 10) - 1, 96 << 10, (96 << 10) + 1, 200_003, 1 << 20):
        p = base[:n]
        want = hash_ref.fold64_c(p) or 1
        assert hash_bytes(p) == want, n
        t = torch.frombuffer(bytearray(p), dtype=torch.uint8).to(cuda)
        assert to_u64_list(hash_tensors([t]))[0] == hash_ref.fold64_c(p), n
    # small-call staging: up to 64 buffers / 64 KiB in one DMA, then the ring path beyond
    for cnt, size in ((64, 1000), (65, 10), (3, 30000), (2, 40000)):
        ps = [base[i * 7:i * 7 + size] for i in range(cnt)]
        assert hash_batch(ps) == [hash_ref.fold64_c(q) for q in ps], (cnt, size)

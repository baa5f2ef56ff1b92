"""Device-counted handshake statistics (SURVEY.md Sec. 8(b) `sesgd_get_stats`): the multi-GPU
kernels count their own cross-GPU flag stores, spins and launches on the device.  On two loopback
virtual ranks (one GPU) the device counts must equal what the protocol prescribes -- the host-side
closed forms (K4 protocol 0: an RS and an AG flag per chunk and remote member; K5: 2(m-1) step
flags per CTA per launch, Eq. 2 / Eq. 3's handshake count) -- and the value-carried protocols must
store no flag at all; sesgd_measure_hop reports a positive one-way hop."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _group(path, protocol, n=2, buckets=(50001, 4099), T=4):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2007_00433_b200 import sesgd as C
    from paper_2007_00433_b200.engine import LoopbackGroup
    opts = {C.OPT_PROTOCOL: protocol} if path == C.PATH_TWOSHOT else {}
    grp = LoopbackGroup(2, n, 2, list(buckets), seed=42, path=path, timeout_ms=10000, options=opts)
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    for e in grp:
        for s, w in enumerate(e.local_workers):
            for b, L in enumerate(buckets):
                synth.fill_x0_device(e.x(s, b).data_ptr(), L, int(offs[b]), e.stream.cuda_stream)
    for t in range(T):
        for e in grp:
            for s, w in enumerate(e.local_workers):
                for b, L in enumerate(buckets):
                    synth.fill_grad_device(e.g(s, b).data_ptr(), L, int(offs[b]), w, t, e.stream.cuda_stream)
        grp.step(t, 0.1, 0.9)
    grp.synchronize()
    grp.poll()
    return grp


def test_k4_flag_protocol_device_counts_match_the_closed_form():
    from paper_2007_00433_b200 import sesgd as C
    grp = _group(C.PATH_TWOSHOT, 0)
    for e in grp:
        st = [e.stats(b) for b in range(2)]
        host = sum(s["flag_messages"] for s in st)
        assert st[0]["dev_flag_stores"] == host > 0, st
        assert st[0]["dev_launches"] == 4 and st[0]["dev_value_spins"] == 0
        assert st[0]["last_launch_us"] > 0
    grp.close()


@pytest.mark.parametrize("protocol", [1, 2])
def test_value_protocols_store_no_flags(protocol):
    from paper_2007_00433_b200 import sesgd as C
    grp = _group(C.PATH_TWOSHOT, protocol)
    for e in grp:
        st = e.stats(0)
        assert st["dev_flag_stores"] == 0 and st["dev_flag_spins"] == 0
        assert st["dev_launches"] == 4
    grp.close()


def test_k5_ring_counts_two_m_minus_one_step_flags_per_cta():
    """Eq. 2 / Eq. 3: a ring allreduce over m members costs 2(m-1) handshakes; K5 stores one step
    flag per CTA per handshake, one launch per bucket and iteration"""
    from paper_2007_00433_b200 import sesgd as C
    grp = _group(C.PATH_RING, 0)
    for e in grp:
        st = [e.stats(b) for b in range(2)]
        assert st[0]["handshake_rounds"] == 2 * (2 - 1)
        assert st[0]["dev_launches"] == 4 * 2
        assert st[0]["dev_flag_stores"] == sum(s["flag_messages"] for s in st) > 0
    grp.close()


def test_measure_hop_between_virtual_ranks():
    from paper_2007_00433_b200 import sesgd as C
    grp = _group(C.PATH_TWOSHOT, 1, T=1)
    a, b = grp[0], grp[1]
    a.measure_hop(1, iters=2000, initiator=True)
    b.measure_hop(0, iters=2000, initiator=False)
    grp.synchronize()
    hop = a.stats(0)["hop_ns"]
    assert 10 < hop < 100000, hop
    grp.close()


@pytest.mark.parametrize("n,mode", [(2, 0), (2, 1), (8, 0), (8, 1)])
def test_k4w_pair_harness_is_bit_exact(n, mode):
    """sesgd_sync_all_pair: both virtual ranks' K4W (n = 2, one worker each) or K4W-M (n = 8, four
    workers each) in one grid (the ncu harness) gives the oracle's bits, like two concurrent launches"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_2007_00433_b200 import sesgd as C
    from paper_2007_00433_b200.engine import LoopbackGroup
    buckets = [100003, 7, 40000]
    grp = LoopbackGroup(2, n, 2, buckets, seed=42, mode=mode, timeout_ms=10000,
                        options={C.OPT_PROTOCOL: 2})
    offs = np.concatenate([[0], np.cumsum(buckets)[:-1]]).astype(np.int64)
    for e in grp:
        for s in range(e.r):
            for b, L in enumerate(buckets):
                synth.fill_x0_device(e.x(s, b).data_ptr(), L, int(offs[b]), e.stream.cuda_stream)
    T = 5
    for t in range(T):
        for e in grp:
            for s, w in enumerate(e.local_workers):
                for b, L in enumerate(buckets):
                    synth.fill_grad_device(e.g(s, b).data_ptr(), L, int(offs[b]), w, t, e.stream.cuda_stream)
        grp.step_pair(t, 0.1, 0.9)
    grp.synchronize()
    grp.poll()
    X = np.stack([torch.cat([e.x(s, b) for b in range(len(buckets))]).cpu().numpy() for e in grp for s in range(e.r)])
    V = np.stack([torch.cat([e.v(s, b) for b in range(len(buckets))]).cpu().numpy() for e in grp for s in range(e.r)])
    assert grp[0].stats(0)["dev_launches"] == T and grp[1].stats(0)["dev_launches"] == T
    grp.close()
    x = np.tile(synth.x0_host(sum(buckets)), (n, 1))
    v = np.zeros_like(x)
    oracle.run(n, 2, 42, T, x, v, s_g=synth.SEED_G, lr=0.1, mu=0.9, mode=mode)
    assert np.array_equal(X.view(np.uint32), x.view(np.uint32))
    assert np.array_equal(V.view(np.uint32), v.view(np.uint32))

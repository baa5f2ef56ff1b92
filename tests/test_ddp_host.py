"""Host logic of SESGDDataParallel's overlap (CPU): bucket readiness and launch order."""
import pytest

from paper_2007_00433_b200.ddp import BucketReadiness


def test_buckets_release_in_order_whatever_the_arrival_order():
    r = BucketReadiness([2, 1, 3])
    assert r.arrive(2) == []           # a later bucket completing first is held back
    assert r.arrive(1) == []
    assert r.arrive(2) == []
    assert r.arrive(0) == []
    assert r.arrive(0) == [0, 1]       # bucket 0 completes -> 0 and the already-complete 1
    assert r.arrive(2) == [2]
    assert r.done()


def test_reset_force_all_and_errors():
    r = BucketReadiness([1, 1])
    assert r.force_all() == [0, 1] and r.done()
    r.reset([1, 1])                    # static-graph trimming: one hook per bucket
    assert not r.done() and r.arrive(1) == [] and r.arrive(0) == [0, 1]
    with pytest.raises(RuntimeError):
        r.arrive(0)                    # more gradients than the bucket holds
    r.reset()
    assert r.release() == [] and not r.done()


def test_empty_bucket_counts_release_immediately():
    r = BucketReadiness([0, 2, 0])
    assert r.release() == [0]
    assert r.arrive(1) == [] and r.arrive(1) == [1, 2]


def test_release_order_property():
    """Any bucket sizes, any arrival order: every bucket is released exactly once, in index order,
    and only after all of its gradients and every earlier bucket's have arrived (the in-order
    launch the per-bucket sync kernels need: buckets are matched across ranks by call order)."""
    from hypothesis import given, settings, strategies as st

    @settings(max_examples=300, deadline=None)
    @given(st.lists(st.integers(0, 4), min_size=1, max_size=8), st.randoms(use_true_random=False))
    def check(counts, rnd):
        arrivals = [b for b, c in enumerate(counts) for _ in range(c)]
        rnd.shuffle(arrivals)
        r = BucketReadiness(counts)
        released = list(r.release())
        seen = [0] * len(counts)
        for b in arrivals:
            seen[b] += 1
            for rb in r.arrive(b):
                assert rb == len(released)                           # in order, once
                assert all(seen[q] == counts[q] for q in range(rb + 1))  # complete, with predecessors
                released.append(rb)
        assert released == list(range(len(counts))) and r.done()

    check()

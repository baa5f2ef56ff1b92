"""CPU tests of bench.py's host-side roofline arithmetic (no GPU, no library).

`nvlink_algo_bytes` is the NVLink term of the roofline bench.py reports for N > 1 (SURVEY.md
Sec. 8(d) d2: a group spanning s GPUs costs each of them 2(s-1)/s * 4 B per element).  Pinned
here to closed forms (two-GPU pair = NCCL's allreduce busbw bytes, full ring over 8 GPUs,
groups resident on one GPU) and to a brute-force recount.
"""
import itertools
import random

import pytest

import bench


def test_pair_across_two_gpus_is_one_copy():
    # n = 2, m = 2, one worker per GPU: each GPU sends (and receives) half the bucket twice.
    assert bench.nvlink_algo_bytes([0, 1], 2, 1, 2, 1000) == 4 * 1000


def test_full_ring_over_eight_gpus():
    # m = n = 8, one worker per GPU: the ring allreduce bound 2 * 7/8 * 4 B per element.
    assert bench.nvlink_algo_bytes(list(range(8)), 8, 1, 8, 1 << 20) == pytest.approx(7 * (1 << 20))


def test_groups_on_one_gpu_cost_nothing():
    # 8 workers resident on one GPU, or each group's members co-resident on one of 4 GPUs.
    assert bench.nvlink_algo_bytes(list(range(8)), 2, 8, 1, 123) == 0.0
    assert bench.nvlink_algo_bytes([0, 1, 2, 3, 4, 5, 6, 7], 2, 2, 4, 123) == 0.0


def test_max_over_gpus():
    # n = 8, m = 2, 2 workers per GPU (4 GPUs): groups {0,2} {1,3} span GPUs 0-1, {4,5} {6,7}
    # are co-resident.  GPUs 0 and 1 each carry two spanning groups: 2 * 4 B * L.
    assert bench.nvlink_algo_bytes([0, 2, 1, 3, 4, 5, 6, 7], 2, 2, 4, 10) == 2 * 4 * 10


def _brute(perm, m, r, world, L):
    # Recount per GPU: for every GPU, every group that has a member there and s distinct GPUs.
    best = 0.0
    for g in range(world):
        tot = 0.0
        for j in range(len(perm) // m):
            gpus = sorted({w // r for w in perm[j * m:(j + 1) * m]})
            if g in gpus:
                tot += (len(gpus) - 1) * 8 * L / len(gpus)
        best = max(best, tot)
    return best


@pytest.mark.parametrize("n,m,world", [(8, 2, 2), (8, 4, 4), (16, 4, 8), (16, 8, 4), (4, 2, 4)])
def test_matches_brute_force_recount(n, m, world):
    rng = random.Random(n * 100 + m * 10 + world)
    r = n // world
    for _ in range(200):
        perm = list(range(n))
        rng.shuffle(perm)
        assert bench.nvlink_algo_bytes(perm, m, r, world, 77) == pytest.approx(_brute(perm, m, r, world, 77))


def test_span_distribution_config3():
    # n = 16, m = 4, 2 workers per GPU on 8 GPUs.  Over all 4-subsets
    # a group spans 4 GPUs with probability C(8,4)*2^4 / C(16,4) = 1120/1820 and 2 GPUs with
    # C(8,2)/C(16,4) = 28/1820; the per-GPU cost of one group is then 6 B or 4 B per element.
    spans = {}
    for grp in itertools.combinations(range(16), 4):
        s = len({w // 2 for w in grp})
        spans[s] = spans.get(s, 0) + 1
    assert spans == {4: 1120, 3: 672, 2: 28}
    # Groups {0,2,4,6} and {1,3,5,7} both span GPUs 0-3 (6 B each there); {8..11}, {12..15}
    # span two GPUs each (4 B): the max is GPU 0..3's 12 B per element.
    assert bench.nvlink_algo_bytes([0, 2, 4, 6] + list(range(8, 16)) + [1, 3, 5, 7], 4, 2, 8, 1) == \
        pytest.approx(12.0)


def test_both_arms_print_the_same_workload():
    """The reference arm (CPU oracle) and the GPU arm name the same config (BASELINE.json cfg 2)."""
    d = bench.workload_desc("resnet50", 8, 2, 5, 25557032, "param")
    assert d == ("cfg2: n=8 workers, group_size=2, resnet50 DDP buckets (5 buckets, 25,557,032 fp32 "
                 "per worker), PARAM mode, lr 0.1, momentum 0.9")


def test_reference_arm_json_workload_equals_gpu_arm_config():
    """The reference arm's emitted config.workload (run here on CPU) is the string the GPU arm
    emits: both come from bench.common_config, and the GPU arm only adds keys beside it."""
    import inspect
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(bench.__file__)
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    d = json.loads(res.stdout.strip().splitlines()[-1])
    want = bench.common_config("resnet50", 8, 2, "param")
    assert d["config"] == {**want, "parallelism": "sesgd groups over 1 GPU(s)"}
    src = inspect.getsource(bench.measure) + inspect.getsource(bench.run_sesgd)
    assert "**common_config(workload, n, m, args.mode)" in src
    assert "workload_desc(" not in src  # nothing appended to the shared string


def test_all_core_oracle_leg_runs_the_plain_oracle_on_every_core():
    """cpu_baseline.all_cores: one unchanged single-threaded oracle per usable core on disjoint
    coordinate subsets; reports the core count and the CPU model beside the number"""
    info = bench.cpu_info()
    assert info["nproc"] >= 1 and info["cpu_count"] >= info["nproc"]
    r = bench.cpu_oracle_all_cores(4, 2, "param", 1 << 20, "config1", rate_1core=2e6, budget_s=0.2)
    assert r["cores"] == info["nproc"] and r["value"] > 0 and r["kind"] == "oracle"


def test_local_groups_on_rank_counts_groups_whose_members_all_live_there():
    """the extra K6 launches of the hybrid K4W-M launch are counted from this host helper:
    worker w lives on rank w // r; a group counts for a rank only if every member lives there"""
    perm = [0, 1, 2, 5, 3, 4, 6, 7]  # canonical groups of m = 2: {0,1} {2,5} {3,4} {6,7}
    assert bench.local_groups_on_rank(perm, 2, 4, 0) == 1  # {0,1}; {2,5} spans ranks 0 and 1
    assert bench.local_groups_on_rank(perm, 2, 4, 1) == 1  # {6,7}
    assert bench.local_groups_on_rank(perm, 2, 2, 1) == 0  # r = 2: rank 1 holds {2, 3}, both partners elsewhere
    assert bench.local_groups_on_rank(perm, 4, 4, 0) == 0  # {0,1,2,5} spans ranks 0 and 1
    assert bench.local_groups_on_rank(list(range(8)), 4, 4, 1) == 1

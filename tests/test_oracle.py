"""The CPU oracle is pinned before it is trusted (CPU-only tests).

Pins: the reference's own known answers (test_core_ops.py, test_datagen.py),
digests of the reference's outputs committed in tests/golden/golden.json, and
-- in the build container only -- a direct comparison with the reference
package including SortStats counters.
"""

import hashlib

import numpy as np
import pytest

from oracle import oracle as O

INT64_MIN = -(2**63)
INT64_MAX = 2**63 - 1


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_mt19937_known_answer(golden):
    # test_datagen.py:62-65
    assert int(O.mt19937_64(5489, 10000)[-1]) == 9981545732273789042
    assert golden["known_answers"]["mt19937_64_seed5489_draw10000"] == 9981545732273789042


def test_first_pass_known_answers(golden):
    kat = golden["known_answers"]
    assert list(O.first_pass(np.array([10, 20, 30, 40]))) == kat["first_pass_10_20_30_40"] == [100, 10, 40]
    assert list(O.first_pass(np.array([INT64_MIN, INT64_MAX]))) == kat["first_pass_extremes"]
    rng = np.random.default_rng(1)
    keys = rng.integers(INT64_MIN, INT64_MAX, size=4096, dtype=np.int64)
    keys[:8] = [INT64_MIN, INT64_MAX, INT64_MIN, INT64_MIN, INT64_MAX, 0, -1, 1]
    s, mn, mx = O.first_pass(keys)
    assert s == sum(int(x) for x in keys) and mn == int(keys.min()) and mx == int(keys.max())


def test_mapping_params_known_answers(golden):
    kat = golden["known_answers"]
    mean, std, zmin, scale = O.mapping_params(np.array([10, 20, 30, 40]), 4)
    assert [mean, std, zmin, scale, 4] == kat["params_10_20_30_40_k4"]
    assert mean == 25.0 and scale == 1.0
    assert [*O.mapping_params(np.array([0, 0, 0, 1]), 2), 2] == kat["params_0_0_0_1_k2"]
    near = np.full(1000, 2**62, np.int64)
    near[::2] += 1
    assert O.mapping_params(near, 8) is None  # DegenerateSpreadError, core.py:229-232
    assert O.cluster_count(10**6, 0.6) == kat["cluster_count_1e6"] == 600


def test_plan_scatter_center_known_answers(golden):
    kat = golden["known_answers"]
    p = kat["params_10_20_30_40_k4"]
    counts = O.histogram(np.array([10, 20, 30, 40]), *p[:4], 4)
    assert [counts.tolist(), [0, 2, 3, 4]] == kat["plan_10_20_30_40"]
    k, c, _ = O.stable_scatter(np.array([10, 40, 10, 30]), np.arange(4), *p[:4], 4)
    assert [k.tolist(), c.tolist()] == kat["scatter_10_40_10_30"]
    assert O.lib().zo_estimated_center(1, p[3], p[2], p[1], p[0]) == kat["estimated_mean_b1"]
    assert O.bucket_of(100, 0.0, 2.0, 0.5, 0.5, 2) == 1 and O.bucket_of(-100, 0.0, 2.0, 0.5, 0.5, 2) == 0


def test_inject_case_matches_reference_digests(golden):
    case = golden["known_answers"]["inject_case"]
    rng = np.random.default_rng(case["seed"])
    keys = rng.integers(-10**12, 10**12, size=case["n"], dtype=np.int64)
    mean, std, zmin, scale = case["params"]
    dk, dc, counts = O.stable_scatter(keys, np.arange(keys.size), mean, std, zmin, scale, case["k"])
    assert counts.tolist() == case["counts"]
    assert sha(dk) == case["scatter_keys_sha"] and sha(dc) == case["scatter_payload_sha"]


@pytest.mark.parametrize("size", [10**3, 10**4, 10**5])
def test_families_match_reference_digests(golden, size):
    for rec in golden["families"]:
        if rec["size"] != size:
            continue
        keys = O.generate_family(rec["kind"], rec["size"], rec["seed"])
        assert sha(keys) == rec["in_keys"], rec
        ok, op, st = O.zsort_ref(keys, np.arange(keys.size, dtype=np.int64))
        assert sha(ok) == rec["keys"] and sha(op) == rec["payload"], rec
        assert st.__dict__ == rec["stats"], rec


def test_adversarial_match_reference_digests(golden):
    two = np.where(np.arange(10**5) % 3 == 0, -7, 123).astype(np.int64)
    ext = np.empty(10**4, np.int64)
    ext[0::2] = INT64_MIN
    ext[1::2] = INT64_MAX
    near = np.full(10**5, 2**62, np.int64)
    near[::2] += 1
    par = O.generate_family("skewed", 10**5, 11, pareto_alpha=1.1)
    cases = {"all_equal": np.full(10**5, 5, np.int64), "two_distinct": two, "extreme_pairs": ext,
             "pareto_1.1": par, "degenerate_spread": near}
    for name, keys in cases.items():
        rec = golden["adversarial"][name]
        assert sha(keys) == rec["in_keys"], name
        ok, op, st = O.zsort_ref(keys, np.arange(keys.size, dtype=np.int64))
        assert sha(ok) == rec["keys"] and sha(op) == rec["payload"], name
        assert st.__dict__ == rec["stats"], name
        assert O.check_stable_permutation(keys, ok, op) == 0


@pytest.mark.parametrize("name", ["C1_n100000", "C2_n100000", "C3_n100000", "C4_n1000000"])
def test_config_variants_match_reference_digests(golden, name):
    rec = golden["configs"][name]
    idx = int(name[1])
    keys, payload = O.make_config(idx, rec["n"])
    assert sha(keys) == rec["in_keys"]
    ok, op, perm = O.stable_sort(keys, payload)
    assert sha(ok) == rec["keys"] and sha(op) == rec["payload"]
    # a stable sort is unique: numpy's stable argsort agrees
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(order, perm)


def test_structural_checker_detects_violations():
    keys = np.array([3, 1, 2, 1], np.int64)
    ok, op, perm = O.stable_sort(keys, None)
    assert O.check_stable_permutation(keys, ok, perm) == 0
    bad = perm.copy()
    bad[0], bad[1] = bad[1], bad[0]  # swap the two equal keys -> unstable
    assert O.check_stable_permutation(keys, ok, bad) >> 56 == 4
    assert O.check_stable_permutation(keys, ok[::-1].copy(), perm[::-1].copy()) >> 56 in (1, 4)
    dup = perm.copy()
    dup[1] = dup[0]
    assert O.check_stable_permutation(keys, ok, dup) >> 56 in (2, 3)


def test_float_keys_zero_and_order():
    keys = np.array([0.0, -0.0, -1.5, 2.0, -0.0, 0.0, -np.inf, np.inf])
    ok, _, perm = O.stable_sort(keys)
    assert np.array_equal(perm, np.argsort(keys, kind="stable"))
    assert np.array_equal(ok.view(np.uint64), keys[perm].view(np.uint64))


@pytest.mark.reference
def test_oracle_equals_reference_including_stats(ref):
    rng = np.random.default_rng(5)
    for trial in range(120):
        kind = O.FAMILIES[trial % 5]
        size = int(rng.integers(1, 20000))
        seed = int(rng.integers(0, 2**63))
        keys = O.generate_family(kind, size, seed)
        assert np.array_equal(keys, ref.generate(ref.DistributionSpec(kind=kind, size=size, seed=seed))[0])
        pay = np.arange(size, dtype=np.int64)
        cfg = {}
        if trial % 7 == 3:
            cfg = dict(alpha=float(rng.uniform(0.1, 2.0)), insertion_threshold=int(rng.integers(1, 200)),
                       counting_range_threshold=int(rng.integers(1, 100000)), depth_guard=int(rng.integers(3, 40)))
        rk, rp, rs = ref.zsort(keys, pay, ref.SortConfig(**cfg) if cfg else None)
        ok, op, os_ = O.zsort_ref(keys, pay, O.OracleConfig(**cfg) if cfg else None)
        assert np.array_equal(rk, ok) and np.array_equal(rp, op), (kind, size, seed)
        assert rs.__dict__ == os_.__dict__, (kind, size, seed)


@pytest.mark.reference
def test_oracle_zsort_rec_equals_reference(ref):
    keys, payload = ref.generate(ref.DistributionSpec(kind="uniform", size=10_000, seed=17))
    center = float(keys.astype(np.float64).mean())
    a = ref.zsort_rec(keys, k=60, scale=15.0, mean_est=center, depth=1, payload=payload)
    b = O.zsort_rec_ref(keys, 60, 15.0, center, 1, payload)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2].__dict__ == b[2].__dict__
    keys, payload = ref.generate(ref.DistributionSpec(kind="skewed", size=5000, seed=3, pareto_alpha=1.1))
    a = ref.zsort_rec(keys, k=40, scale=10.0, mean_est=1e18, payload=payload)
    b = O.zsort_rec_ref(keys, 40, 10.0, 1e18, 1, payload)
    assert np.array_equal(a[0], b[0]) and a[2].__dict__ == b[2].__dict__

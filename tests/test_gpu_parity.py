"""GPU parity: the CUDA path through the C ABI against the CPU oracle and the
committed reference digests.  Bit-exact for keys and payload permutation.

Mirrors the reference's own tests (pkg/tests/test_zsort.py,
test_core_ops.py, test_acceptance.py criteria 1 and 5) with the GPU
implementation swapped in, plus the BASELINE.json configs.
"""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

INT64_MIN = -(2**63)
INT64_MAX = 2**63 - 1


@pytest.fixture(scope="module")
def Z():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_14419_b200 as Z
    return Z


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def assert_matches_oracle(Z, keys, payload=None, config=None):
    keys = np.ascontiguousarray(keys)
    if payload is None:
        payload = np.arange(keys.size, dtype=np.int64)
    ok, op, st = Z.zsort(keys, payload, config)
    ek, ep, _ = O.stable_sort(keys, payload)
    assert ok.dtype == keys.dtype
    np.testing.assert_array_equal(ok.view(np.uint64), ek.view(np.uint64))
    np.testing.assert_array_equal(op, ep)
    return ok, op, st


# ------------------------------------------------ reference unit tests

class TestBasics:  # test_zsort.py:36-86
    def test_empty(self, Z):
        k, p, s = Z.zsort(np.array([], np.int64))
        assert k.size == 0 and p is None and s.total_scatter_passes == 0

    def test_thousand_records_hundred_distinct(self, Z):
        keys = np.random.default_rng(0).integers(0, 100, size=1000, dtype=np.int64)
        assert_matches_oracle(Z, keys)

    def test_all_equal_copies_through(self, Z):
        keys = np.full(10**5, 77, np.int64)
        k, p, s = Z.zsort(keys, np.arange(10**5))
        assert np.array_equal(k, keys) and np.array_equal(p, np.arange(10**5))
        assert s.max_depth_reached == 0 and s.total_scatter_passes == 0

    def test_small_input(self, Z):
        k, p, s = Z.zsort(np.array([5, 1, 5, -2], np.int64), np.arange(4))
        assert k.tolist() == [-2, 1, 5, 5] and p.tolist() == [3, 1, 0, 2]
        assert s.total_scatter_passes == 0 and s.insertion_sort_invocations == 1

    def test_inputs_untouched(self, Z):
        keys = np.array([9, 2, 7, 2] * 100, np.int64)
        payload = np.arange(keys.size, dtype=np.int64)
        kc, pc = keys.copy(), payload.copy()
        Z.zsort(keys, payload)
        assert np.array_equal(keys, kc) and np.array_equal(payload, pc)
        tk = torch.from_numpy(O.generate_family("uniform", 50_000, 3)).cuda()
        tc = tk.clone()
        Z.zsort(tk)
        assert torch.equal(tk, tc)

    def test_determinism(self, Z):
        keys = O.generate_family("normal", 50_000, 8)
        a = Z.zsort(keys, np.arange(keys.size))
        b = Z.zsort(keys, np.arange(keys.size))
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])

    def test_payload_mismatch(self, Z):
        with pytest.raises(ValueError):
            Z.zsort(np.array([1, 2], np.int64), payload=np.arange(3))

    def test_nan_keys_rejected(self, Z):
        keys = np.random.default_rng(1).standard_normal(20_000)
        keys[777] = np.nan
        with pytest.raises(ValueError):
            Z.zsort(keys)


class TestPayloadModes:  # test_zsort.py:214-240
    def test_none_payload(self, Z):
        k, p, _ = Z.zsort(np.array([3, 1, 2], np.int64))
        assert p is None and k.tolist() == [1, 2, 3]

    def test_uint64_payload_by_view(self, Z):
        k, p, _ = Z.zsort(np.array([2, 1, 2, 1], np.int64), np.array([10, 11, 12, 13], np.uint64))
        assert p.dtype == np.uint64 and p.tolist() == [11, 13, 10, 12]

    def test_float_payload_bit_exact(self, Z):
        k, p, _ = Z.zsort(np.array([5, -5], np.int64), np.array([np.nan, 2.5]))
        assert k.tolist() == [-5, 5] and p[0] == 2.5 and np.isnan(p[1])

    def test_wide_payload_gathers_by_index(self, Z):
        keys = np.array([4, 2, 4, 2] * 50, np.int64)
        payload = np.array([f"rec{i}" for i in range(200)], dtype="U8")
        k, p, _ = Z.zsort(keys, payload)
        ek, ep, _ = O.stable_sort(keys, payload)
        assert np.array_equal(k, ek) and np.array_equal(p, ep)

    @pytest.mark.parametrize("dt", [np.int32, np.float32, np.uint32, np.int16, np.int64])
    def test_payload_dtypes_large(self, Z, dt):
        keys = O.generate_family("normal", 100_000, 4)
        payload = (np.arange(keys.size) % 30000).astype(dt)
        assert_matches_oracle(Z, keys, payload)

    def test_torch_cuda_roundtrip(self, Z):
        keys = O.generate_family("skewed", 200_000, 9)
        tk = torch.from_numpy(keys).cuda()
        tp = torch.arange(keys.size, dtype=torch.int32, device="cuda")
        k, p, _ = Z.zsort(tk, tp)
        assert k.is_cuda and p.is_cuda and p.dtype == torch.int32
        ek, ep, _ = O.stable_sort(keys, np.arange(keys.size, dtype=np.int32))
        assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(p.cpu().numpy(), ep)


class TestBuildingBlocks:  # test_core_ops.py with K1/K2/K4 parameter injection
    def test_first_pass_known_answers(self, Z, golden):
        kat = golden["known_answers"]
        st = Z.first_pass(np.array([10, 20, 30, 40], np.int64))
        assert [st.sum, st.min_key, st.max_key] == kat["first_pass_10_20_30_40"]
        st = Z.first_pass(np.array([INT64_MIN, INT64_MAX], np.int64))
        assert [st.sum, st.min_key, st.max_key] == kat["first_pass_extremes"]
        rng = np.random.default_rng(1)
        keys = rng.integers(INT64_MIN, INT64_MAX, size=1 << 20, dtype=np.int64)
        keys[:8] = [INT64_MIN, INT64_MAX, INT64_MIN, INT64_MIN, INT64_MAX, 0, -1, 1]
        st = Z.first_pass(keys)
        assert st.sum == sum(int(x) for x in keys[:1000]) + sum(int(x) for x in keys[1000:]) or True
        assert st.sum == int(np.sum(keys.astype(object)))
        assert st.min_key == int(keys.min()) and st.max_key == int(keys.max())

    def test_mapping_params(self, Z, golden):
        kat = golden["known_answers"]
        keys = np.array([10, 20, 30, 40], np.int64)
        p = Z.build_mapping_params(keys, Z.first_pass(keys), 4)
        ref = kat["params_10_20_30_40_k4"]
        assert p.mean == ref[0] and p.scale == ref[3] and p.k == 4
        assert p.std == pytest.approx(ref[1], rel=1e-15) and p.zmin == pytest.approx(ref[2], rel=1e-15)
        near = np.full(1000, 2**62, np.int64)
        near[::2] += 1
        with pytest.raises(Z.DegenerateSpreadError):
            Z.build_mapping_params(near, Z.first_pass(near), 8)
        # one-pass fp64 variance agrees with the sequential two-pass oracle
        rng = np.random.default_rng(7)
        keys = rng.integers(-10**15, 10**15, size=200_000, dtype=np.int64)
        p = Z.build_mapping_params(keys, Z.first_pass(keys), 32)
        mean, std, zmin, scale = O.mapping_params(keys, 32)
        assert p.mean == mean and p.scale == scale
        assert p.std == pytest.approx(std, rel=1e-12) and p.zmin == pytest.approx(zmin, rel=1e-12)

    def test_plan_and_scatter_known_answers(self, Z, golden):
        kat = golden["known_answers"]
        r = kat["params_10_20_30_40_k4"]
        params = Z.MappingParams(mean=r[0], std=r[1], zmin=r[2], scale=r[3], k=4)
        plan = Z.build_partition_plan(np.array([10, 20, 30, 40], np.int64), params)
        assert [plan.counts.tolist(), plan.offsets.tolist()] == kat["plan_10_20_30_40"]
        src = np.array([10, 40, 10, 30], np.int64)
        k, c = Z.stable_scatter(src, Z.build_partition_plan(src, params), params, np.arange(4, dtype=np.int64))
        assert [k.tolist(), c.tolist()] == kat["scatter_10_40_10_30"]
        assert Z.map_to_cluster(100, Z.MappingParams(0.0, 2.0, 0.5, 0.5, 2)) == 1
        assert Z.map_to_cluster(-100, Z.MappingParams(0.0, 2.0, 0.5, 0.5, 2)) == 0
        assert Z.estimated_mean(1, params) == kat["estimated_mean_b1"]

    def test_injected_params_match_reference(self, Z, golden):
        case = golden["known_answers"]["inject_case"]
        rng = np.random.default_rng(case["seed"])
        keys = rng.integers(-10**12, 10**12, size=case["n"], dtype=np.int64)
        mean, std, zmin, scale = case["params"]
        params = Z.MappingParams(mean, std, zmin, scale, case["k"])
        plan = Z.build_partition_plan(keys, params)
        assert plan.counts.tolist() == case["counts"]
        k, c = Z.stable_scatter(keys, plan, params, np.arange(keys.size, dtype=np.int64))
        assert sha(k) == case["scatter_keys_sha"] and sha(c) == case["scatter_payload_sha"]

    @pytest.mark.parametrize("n,k", [(10**6, 600), (3 * 10**6, 2048), (10**6, 1500)])
    def test_large_injected_scatter_vs_oracle(self, Z, n, k):
        keys = O.generate_family("normal", n, 21)
        mean, std, zmin, scale = O.mapping_params(keys, k)
        params = Z.MappingParams(mean, std, zmin, scale, k)
        plan = Z.build_partition_plan(keys, params)
        assert plan.counts.tolist() == O.histogram(keys, mean, std, zmin, scale, k).tolist()
        gk, gc = Z.stable_scatter(keys, plan, params, np.arange(n, dtype=np.int64))
        ek, ec, _ = O.stable_scatter(keys, np.arange(n), mean, std, zmin, scale, k)
        assert np.array_equal(gk, ek) and np.array_equal(gc, ec)


    # fan-outs <= 32 rank by the register multi-split (ballots, no shared
    # atomics); 33 and 64 take the shared-atomic path with the tie-group loop
    @pytest.mark.parametrize("k", [2, 3, 16, 17, 31, 32, 33, 64])
    @pytest.mark.parametrize("kind,n", [("normal", 1_000_003), ("sorted", 300_017), ("few", 50_001), ("normal", 4099)])
    def test_small_fanout_scatter_vs_oracle(self, Z, k, kind, n):
        rng = np.random.default_rng(k * 1000 + n % 997)
        if kind == "normal":
            keys = (rng.standard_normal(n) * 1e9).astype(np.int64)
        elif kind == "sorted":  # whole rows of lanes in one bucket, a few displaced records
            keys = np.sort(rng.integers(-10**12, 10**12, size=n, dtype=np.int64))
            sw = rng.integers(0, n, size=(n // 50, 2))
            keys[sw[:, 0]], keys[sw[:, 1]] = keys[sw[:, 1]].copy(), keys[sw[:, 0]].copy()
        else:
            keys = rng.choice(np.array([-7, 0, 5, 10**9, -10**9], np.int64), size=n)
        mean, std, zmin, scale = O.mapping_params(keys, k)
        params = Z.MappingParams(mean, std, zmin, scale, k)
        plan = Z.build_partition_plan(keys, params)
        assert plan.counts.tolist() == O.histogram(keys, mean, std, zmin, scale, k).tolist()
        gk, gc = Z.stable_scatter(keys, plan, params, np.arange(n, dtype=np.int64))
        ek, ec, _ = O.stable_scatter(keys, np.arange(n), mean, std, zmin, scale, k)
        assert np.array_equal(gk, ek) and np.array_equal(gc, ec)


# ------------------------------------------------ end to end vs oracle

@pytest.mark.parametrize("mapping", ["fitted", "paper"])
class TestFamilies:
    def test_acceptance_criterion_1_instances(self, Z, golden, mapping):
        cfg = Z.SortConfig(mapping=mapping)
        for rec in golden["families"]:
            keys = O.generate_family(rec["kind"], rec["size"], rec["seed"])
            assert sha(keys) == rec["in_keys"]
            k, p, _ = Z.zsort(keys, np.arange(keys.size, dtype=np.int64), cfg)
            assert sha(k) == rec["keys"] and sha(p) == rec["payload"], (rec["kind"], rec["size"], rec["seed"])

    def test_adversarial_criterion_5(self, Z, golden, mapping):
        cfg = Z.SortConfig(mapping=mapping)
        two = np.where(np.arange(10**5) % 3 == 0, -7, 123).astype(np.int64)
        ext = np.empty(10**4, np.int64)
        ext[0::2] = INT64_MIN
        ext[1::2] = INT64_MAX
        near = np.full(10**5, 2**62, np.int64)
        near[::2] += 1
        cases = {"all_equal": np.full(10**5, 5, np.int64), "two_distinct": two, "extreme_pairs": ext,
                 "pareto_1.1": O.generate_family("skewed", 10**5, 11, pareto_alpha=1.1), "degenerate_spread": near}
        for name, keys in cases.items():
            rec = golden["adversarial"][name]
            k, p, _ = Z.zsort(keys, np.arange(keys.size, dtype=np.int64), cfg)
            assert sha(k) == rec["keys"] and sha(p) == rec["payload"], name

    def test_randomized_instances(self, Z, mapping):  # test_zsort.py:128-148
        rng = np.random.default_rng(2024)
        cfg = Z.SortConfig(mapping=mapping)
        for trial in range(150):
            kind = O.FAMILIES[trial % 5]
            size = int(rng.integers(1, 60_000))
            seed = int(rng.integers(0, 2**63))
            keys = O.generate_family(kind, size, seed)
            assert_matches_oracle(Z, keys, None, cfg)

    def test_medium_generators_no_fallback(self, Z, mapping):  # test_zsort.py:117-126
        for kind in O.FAMILIES:
            keys = O.generate_family(kind, 20_000, 31)
            k, p, s = Z.zsort(keys, np.arange(keys.size), Z.SortConfig(mapping=mapping))
            ek, ep, _ = O.stable_sort(keys, np.arange(keys.size))
            assert np.array_equal(k, ek) and np.array_equal(p, ep)
            assert s.fallback_invocations == 0, kind


class TestEdgeCases:
    @pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 95, 96, 97, 4095, 4096, 4097, 8191, 8192, 8193, 12345,
                                   65535, 65536, 65537])
    def test_ragged_sizes(self, Z, n):
        rng = np.random.default_rng(n)
        assert_matches_oracle(Z, rng.integers(-50, 50, size=n, dtype=np.int64))
        assert_matches_oracle(Z, rng.integers(INT64_MIN, INT64_MAX, size=n, endpoint=True, dtype=np.int64))
        assert_matches_oracle(Z, rng.standard_normal(n))

    def test_float_signed_zeros_and_infinities(self, Z):
        rng = np.random.default_rng(3)
        keys = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, 5e-324, -5e-324, 1e308]), 300_000)
        assert_matches_oracle(Z, keys)
        assert_matches_oracle(Z, keys[:50])

    def test_presorted_reversed_and_sawtooth(self, Z):
        n = 1_000_000
        asc = np.arange(n, dtype=np.int64) * 7919
        assert_matches_oracle(Z, asc)
        assert_matches_oracle(Z, asc[::-1].copy())
        assert_matches_oracle(Z, (np.arange(n) % 1000).astype(np.int64))

    def test_clustered_with_outliers(self, Z):
        rng = np.random.default_rng(5)
        keys = rng.integers(0, 100, size=500_000, dtype=np.int64)
        keys[::50_000] = INT64_MAX - rng.integers(0, 5, size=10)
        keys[1::70_000] = INT64_MIN
        assert_matches_oracle(Z, keys)
        f = rng.standard_normal(500_000) * 1e-300
        f[::1000] = 1e300
        assert_matches_oracle(Z, f)

    def test_sample_blind_spots(self, Z):
        # The fitted level 1 maps from a stratified sample (runs of 32 keys every
        # n/8192 positions).  Keys that agree on every sampled position but not
        # elsewhere force the exact fallback; a NaN outside the sample must
        # still be rejected (K2 screens every key).
        n = 1 << 20
        stride = n // 8192
        pos = np.arange(n)
        sampled = (pos % stride) < 32
        rng = np.random.default_rng(11)
        keys = np.where(sampled, 0, rng.integers(-10**6, 10**6, size=n)).astype(np.int64)
        assert_matches_oracle(Z, keys)
        f = np.where(sampled, 1.5, rng.standard_normal(n))
        assert_matches_oracle(Z, f)
        g = rng.standard_normal(n)
        g[np.flatnonzero(~sampled)[12345]] = np.nan
        with pytest.raises(ValueError):
            Z.zsort(g)

    def test_nondefault_thresholds(self, Z):  # test_zsort.py:107-114
        keys = np.random.default_rng(42).integers(-10**10, 10**10, size=50_000, dtype=np.int64)
        for cfg in (Z.SortConfig(insertion_threshold=1, counting_range_threshold=1), Z.SortConfig(depth_guard=3),
                    Z.SortConfig(alpha=0.1, mapping="paper"), Z.SortConfig(alpha=2.0, mapping="paper")):
            assert_matches_oracle(Z, keys, None, cfg)

    def test_device_structural_checker(self, Z):
        keys = O.generate_family("high_duplicate", 300_000, 4)
        tk = torch.from_numpy(keys).cuda()
        idx = torch.arange(keys.size, dtype=torch.int64, device="cuda")
        k, p, _ = Z.zsort(tk, idx)
        assert Z.check_stable_permutation_device(tk, k, p) == 0
        bad = p.clone()
        j = int(torch.nonzero(k[1:] == k[:-1])[0]) if bool((k[1:] == k[:-1]).any()) else 0
        bad[j], bad[j + 1] = p[j + 1], p[j]
        assert Z.check_stable_permutation_device(tk, k, bad) > 0


# ------------------------------------------------ BASELINE.json configs

@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C1_n100000", "C2_n100000", "C3_n100000", "C4_n1000000"])
def test_baseline_configs_match_reference_digests(Z, golden, name):
    rec = golden["configs"][name]
    keys, payload = O.make_config(int(name[1]), rec["n"])
    assert sha(keys) == rec["in_keys"]
    k, p, _ = Z.zsort(keys, payload)
    assert sha(k) == rec["keys"] and sha(p) == rec["payload"], name


def test_config4_full_matches_reference_digest(Z, golden):
    rec = golden["configs"]["C4"]
    keys, payload = O.make_config(4, rec["n"])
    assert sha(keys) == rec["in_keys"]
    for mapping in ("fitted", "paper"):
        k, p, _ = Z.zsort(keys, payload, Z.SortConfig(mapping=mapping))
        assert sha(k) == rec["keys"] and sha(p) == rec["payload"], mapping


def test_config5_shape_structural_single_gpu(Z):
    """Config 5 recipe (uniform int64 with a 10% repeated value, int64 index
    payload) at 2^26 on one GPU: device structural check + host oracle."""
    from paper_2605_14419_b200 import datagen
    n = 1 << 26
    keys = datagen.config5_keys(0, n, n, device="cuda")
    idx = torch.arange(n, dtype=torch.int64, device="cuda")
    k, p, _ = Z.zsort(keys, idx)
    assert Z.check_stable_permutation_device(keys, k, p) == 0
    hk = keys[: 1 << 22].cpu().numpy()
    ok, op, _ = Z.zsort(hk, np.arange(hk.size, dtype=np.int64))
    ek, ep, _ = O.stable_sort(hk, np.arange(hk.size, dtype=np.int64))
    assert np.array_equal(ok, ek) and np.array_equal(op, ep)


# ------------------------------------------------ bench seam

def test_harness_seam(Z):
    from paper_2605_14419_b200 import harness

    registry = {}
    name = harness.register(lambda n, a: registry.__setitem__(n, a))
    keys = O.generate_family("uniform", 50_000, 9)
    pay = np.arange(keys.size, dtype=np.int64)[::-1].copy()
    k, p = registry[name](keys.copy(), pay.copy(), None)
    ek, ep, _ = O.stable_sort(keys, pay)
    assert np.array_equal(k, ek) and np.array_equal(p, ep)
    r = harness.run_trial_gpu(keys, pay.astype(np.int32), repetitions=3)
    assert r.verified and r.size == keys.size and r.min_ms > 0


@pytest.mark.parametrize("kind", ["lognormal", "sorted_swaps", "steps"])
def test_two_levels_with_small_children(Z, kind):
    # float64 keys, int32 payload, sized so level 1 leaves children of 2-32
    # buckets: their scatter ranks by the register multi-split
    rng = np.random.default_rng(11)
    n = 3_000_001
    if kind == "lognormal":
        keys = rng.lognormal(0.0, 2.0, n)
    elif kind == "sorted_swaps":
        keys = np.sort(rng.random(n) * 1e6)
        sw = rng.integers(0, n, size=(n // 100, 2))
        keys[sw[:, 0]], keys[sw[:, 1]] = keys[sw[:, 1]].copy(), keys[sw[:, 0]].copy()
        keys[: n // 2] = rng.lognormal(0.0, 2.0, n // 2)
    else:  # long runs of equal keys between random stretches
        keys = np.repeat(rng.standard_normal(n // 1000 + 1), 1000)[:n] + (rng.random(n) < 0.5) * rng.standard_normal(n)
    pay = np.arange(n, dtype=np.int32)
    k, p, st = Z.zsort(keys, pay)
    ek, ep, _ = O.stable_sort(keys, pay)
    assert np.array_equal(k.view(np.uint64), ek.view(np.uint64)) and np.array_equal(p, ep)
    if kind == "lognormal":
        assert st.max_depth_reached >= 2


def test_scatter_tie_groups(Z):
    # the scatter ranks items with shared atomics; lanes of one instruction
    # that share a bucket (tie groups) are detected on every instruction and
    # re-ranked in lane order, so stability does not rest on the hardware's
    # order of atomic results
    rng = np.random.default_rng(77)
    few = rng.integers(0, 50, size=2_000_000).astype(np.int64)
    assert_matches_oracle(Z, few)
    runs = np.repeat(rng.standard_normal(20_000), 100)  # sorted-run-like ties inside warps
    assert_matches_oracle(Z, runs)
    two = rng.integers(0, 2, size=3_000_000).astype(np.int64) << 40  # two buckets: every lane ties
    assert_matches_oracle(Z, two)


def _nested_scales(rng, n, levels, outliers=12):
    """Keys whose range is stretched by a few outliers at every scale: the
    bulk of each finish run lands in one sub-bucket (an oversized digit), and
    the refine run of that digit is stretched again by the next scale's
    outliers, so refine runs produce refine runs (the device ping-pong)."""
    keys = rng.integers(0, 1000, size=n, dtype=np.int64)
    pos = rng.permutation(n)
    at = 0
    for lv in range(levels):
        scale = 10 ** (3 * (lv + 1))
        sel = pos[at:at + outliers]
        keys[sel] = rng.integers(scale, min(10 * scale, 2**62), size=sel.size, dtype=np.int64)
        at += outliers
    return keys


@pytest.mark.parametrize("n,levels", [(12000, 5), (8000, 6), (200_000, 5), (3_000_000, 4)])
def test_nested_refine_runs(Z, n, levels):
    rng = np.random.default_rng(1000 + levels)
    keys = _nested_scales(rng, n, levels)
    ok, op, st = assert_matches_oracle(Z, keys)
    if n <= 12000:  # one shared-memory finish: every further run is a refine run
        assert st.insertion_sort_invocations > 2, st


def test_stream_ordered_without_stats(Z):
    """zsb_sort with no stats buffer returns once the sort is enqueued; after a
    stream sync the output equals the synchronous call's."""
    import ctypes
    from paper_2605_14419_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(77)
    keys = torch.from_numpy(rng.standard_normal(3_000_000)).cuda()
    pay = torch.arange(keys.numel(), dtype=torch.int32, device="cuda")
    c = Z.SortConfig().to_c()
    n = keys.numel()
    ws_bytes = L.zsb_workspace_bytes(n, 1, 4, c)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    outs = []
    for with_stats in (True, False):
        ok, op = torch.empty_like(keys), torch.empty_like(pay)
        stats = (ctypes.c_int64 * 5)() if with_stats else None
        rc = L.zsb_sort(keys.data_ptr(), 1, pay.data_ptr(), 4, ok.data_ptr(), op.data_ptr(), n, c, ws.data_ptr(),
                        ws_bytes, stats, torch.cuda.current_stream().cuda_stream)
        _lib.check(rc)
        torch.cuda.current_stream().synchronize()
        outs.append((ok.cpu().numpy(), op.cpu().numpy()))
    assert np.array_equal(outs[0][0].view(np.uint64), outs[1][0].view(np.uint64))
    assert np.array_equal(outs[0][1], outs[1][1])
    ek, ep, _ = O.stable_sort(keys.cpu().numpy(), pay.cpu().numpy())
    assert np.array_equal(outs[1][1], ep)

"""On-device family generator (zsb_generate, csrc/gen_kernels.cuh) against
the shapes of the reference's families (datagen.py:92-162), and the sort of
each family: small sizes against the CPU oracle, 10^8 keys through the device
structural checker (sorted + permutation + key match + stability)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Z():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_14419_b200 as Z
    return Z


def test_counter_based_and_shardable(Z):
    from paper_2605_14419_b200.datagen import FAMILIES, device_family

    for kind in FAMILIES:
        whole = device_family(kind, 1 << 16, seed=5)
        again = device_family(kind, 1 << 16, seed=5)
        assert torch.equal(whole, again), kind  # a pure function of (family, seed, i)
        part = device_family(kind, 1000, seed=5, offset=20_000, n_total=1 << 16)
        assert torch.equal(part, whole[20_000:21_000]), kind  # any shard regenerates its keys
        assert not torch.equal(whole, device_family(kind, 1 << 16, seed=6)), kind


def test_family_shapes(Z):
    from paper_2605_14419_b200.datagen import device_family

    n = 1 << 22
    u = device_family("uniform", n).cpu().numpy()
    assert abs(u.astype(np.float64).mean()) < 2**63 * 0.01 and u.min() < -(2**62) and u.max() > 2**62
    z = device_family("normal", n).cpu().numpy().astype(np.float64)
    assert abs(z.mean()) < 3e6 and abs(z.std() / 1e9 - 1.0) < 0.01  # mu 0, sigma 1e9
    assert np.all(z == np.rint(z))
    s = device_family("skewed", n).cpu().numpy()
    assert s.min() == 1  # floor(xm * u^(-1/alpha)) >= xm = 1
    med = np.median(s.astype(np.float64))
    assert med == np.floor(2 ** (1 / 1.5))  # Pareto(1.5) median 2^(1/alpha) = 1.587 -> 1
    assert (s >= 10).mean() == pytest.approx(10 ** -1.5, rel=0.05)
    ns = device_family("nearly_sorted", n).cpu().numpy()
    ordered = np.mean(ns[1:] >= ns[:-1])
    assert 0.95 < ordered < 0.995  # a sorted run with ~2% displaced positions
    h = device_family("high_duplicate", n).cpu().numpy()
    assert h.min() == 0 and h.max() == 999 and np.unique(h).size == 1000


@pytest.mark.parametrize("kind", ["uniform", "normal", "skewed", "nearly_sorted", "high_duplicate"])
def test_family_sort_matches_oracle(Z, kind):
    from oracle import oracle as O
    from paper_2605_14419_b200.datagen import device_family

    keys = device_family(kind, 300_000, seed=11).cpu().numpy()
    pay = np.arange(keys.size, dtype=np.int32)
    k, p, _ = Z.zsort(keys, pay)
    ek, ep, _ = O.stable_sort(keys, pay)
    assert np.array_equal(k, ek) and np.array_equal(p, ep)


@pytest.mark.parametrize("kind", ["uniform", "normal", "skewed", "nearly_sorted", "high_duplicate"])
def test_family_sort_1e8_device_check(Z, kind):
    from paper_2605_14419_b200.datagen import device_family

    n = 10**8
    keys = device_family(kind, n, seed=3)
    idx = torch.arange(n, dtype=torch.int32, device="cuda")
    k, p, st = Z.zsort(keys, idx)
    assert Z.check_stable_permutation_device(keys, k, p) == 0, kind
    assert st.fallback_invocations == 0 or kind == "high_duplicate"

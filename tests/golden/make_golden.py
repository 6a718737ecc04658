"""Generate tests/golden/golden.json from the REFERENCE implementation.

Run in the build container, where the reference package is importable from
/root/reference/pkg/src (it does not exist on the GPU box, which is why the
outputs are committed as digests):

    python tests/golden/make_golden.py

Every digest is SHA-256 over the little-endian bytes of the reference's own
``zsort`` output (sorted keys, and the payload permutation it carried).  Float
configs go through the reference as their order-preserving int64 image with
the original index as payload, and the float keys are gathered
back by that permutation.  Inputs are digested too, so a generator drift on
the GPU box is caught before any sort is compared.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import zsort as REF  # noqa: E402  (the reference package, read-only)

from oracle import oracle as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_sort_any(keys: np.ndarray, payload: np.ndarray):
    """Reference zsort on int64 keys, or on the f2i image for float64."""
    if keys.dtype == np.float64:
        img = O.f2i(keys)
        _, perm, stats = REF.zsort(img, np.arange(keys.size, dtype=np.int64))
        return keys[perm], payload[perm], stats
    return REF.zsort(keys, payload)


def stats_dict(s) -> dict:
    return {k: int(v) for k, v in s.__dict__.items()}


def main():
    out = {"generated_by": "tests/golden/make_golden.py", "reference": "/root/reference/pkg/src/zsort"}

    # -- known-answer vectors pinned by the reference's unit tests --------
    kat = {}
    kat["mt19937_64_seed5489_draw10000"] = int(REF.datagen.fill_raw(5489, 10000)[-1])  # test_datagen.py:62-65
    fp = REF.first_pass(np.array([10, 20, 30, 40], np.int64))
    kat["first_pass_10_20_30_40"] = [fp.sum, fp.min_key, fp.max_key]
    fp = REF.first_pass(np.array([-(2**63), 2**63 - 1], np.int64))
    kat["first_pass_extremes"] = [fp.sum, fp.min_key, fp.max_key]
    keys4 = np.array([10, 20, 30, 40], np.int64)
    p = REF.build_mapping_params(keys4, REF.first_pass(keys4), 4)
    kat["params_10_20_30_40_k4"] = [p.mean, p.std, p.zmin, p.scale, p.k]
    plan = REF.build_partition_plan(keys4, p)
    kat["plan_10_20_30_40"] = [plan.counts.tolist(), plan.offsets.tolist()]
    sk, sp = REF.stable_scatter(np.array([10, 40, 10, 30], np.int64), REF.build_partition_plan(
        np.array([10, 40, 10, 30], np.int64), p), p, np.arange(4, dtype=np.int64))
    kat["scatter_10_40_10_30"] = [sk.tolist(), sp.tolist()]
    kat["estimated_mean_b1"] = REF.estimated_mean(1, p)
    kat["cluster_count_1e6"] = REF.cluster_count(10**6, 0.6)
    p01 = REF.build_mapping_params(np.array([0, 0, 0, 1], np.int64), REF.first_pass(np.array([0, 0, 0, 1])), 2)
    kat["params_0_0_0_1_k2"] = [p01.mean, p01.std, p01.zmin, p01.scale, p01.k]
    # random param-injection case for the K2/K4 kernel-level parity tests
    rng = np.random.default_rng(11)
    kr = rng.integers(-10**12, 10**12, size=4099, dtype=np.int64)
    pr = REF.build_mapping_params(kr, REF.first_pass(kr), 37)
    planr = REF.build_partition_plan(kr, pr)
    skr, spr = REF.stable_scatter(kr, planr, pr, np.arange(kr.size, dtype=np.int64))
    kat["inject_case"] = {
        "seed": 11, "n": 4099, "k": 37, "params": [pr.mean, pr.std, pr.zmin, pr.scale],
        "counts": planr.counts.tolist(), "scatter_keys_sha": sha(skr), "scatter_payload_sha": sha(spr),
    }
    out["known_answers"] = kat

    # -- acceptance criterion 1 instances (test_acceptance.py:67-87) ------
    fam = []
    t0 = time.time()
    for kind in ("uniform", "normal", "skewed", "nearly_sorted", "high_duplicate"):
        for size in (10**3, 10**4, 10**5, 10**6):
            for seed in (101, 202, 303):
                keys, payload = REF.generate(REF.DistributionSpec(kind=kind, size=size, seed=seed))
                ok, op, st = REF.zsort(keys, payload)
                fam.append({"kind": kind, "size": size, "seed": seed, "in_keys": sha(keys),
                            "keys": sha(ok), "payload": sha(op), "stats": stats_dict(st)})
    out["families"] = fam
    print(f"families: {len(fam)} in {time.time() - t0:.1f}s", flush=True)

    # -- adversarial inputs, acceptance criterion 5 (test_acceptance.py:152-180)
    adv = {}
    two = np.where(np.arange(10**5) % 3 == 0, -7, 123).astype(np.int64)
    ext = np.empty(10**4, np.int64)
    ext[0::2] = -(2**63)
    ext[1::2] = 2**63 - 1
    near = np.full(10**5, 2**62, np.int64)
    near[::2] += 1
    par = REF.generate(REF.DistributionSpec(kind="skewed", size=10**5, seed=11, pareto_alpha=1.1))[0]
    for name, keys in {"all_equal": np.full(10**5, 5, np.int64), "two_distinct": two, "extreme_pairs": ext,
                       "pareto_1.1": par, "degenerate_spread": near}.items():
        ok, op, st = REF.zsort(keys, np.arange(keys.size, dtype=np.int64))
        adv[name] = {"in_keys": sha(keys), "keys": sha(ok), "payload": sha(op), "stats": stats_dict(st)}
    out["adversarial"] = adv

    # -- BASELINE configs 1..4 at full size, plus scaled-down variants ----
    cfgs = {}
    for idx, sizes in ((1, (None, 10**5)), (2, (None, 10**5)), (3, (None, 10**5)), (4, (None, 10**6))):
        for n in sizes:
            t0 = time.time()
            keys, payload = O.make_config(idx, n)
            ok, op, st = ref_sort_any(keys, payload)
            name = f"C{idx}" + ("" if n is None else f"_n{n}")
            cfgs[name] = {"n": int(keys.size), "dtype": str(keys.dtype), "in_keys": sha(keys),
                          "keys": sha(ok), "payload": sha(op), "stats": stats_dict(st)}
            print(f"{name}: reference sorted {keys.size} in {time.time() - t0:.1f}s", flush=True)
    out["configs"] = cfgs

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote golden.json")


if __name__ == "__main__":
    main()

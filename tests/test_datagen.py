"""Workload recipes used by bench.py (paper_2605_14419_b200/datagen.py) must
produce exactly the inputs the reference digests were computed on
(tests/golden/golden.json, made by tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from paper_2605_14419_b200 import datagen


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["C1", "C1_n100000", "C2_n100000", "C3_n100000", "C4_n1000000"])
def test_baseline_config_inputs_match_reference_digests(golden, name):
    rec = golden["configs"][name]
    keys, payload = datagen.baseline_config(int(name[1]), rec["n"])
    assert keys.size == rec["n"] and sha(keys) == rec["in_keys"]
    assert np.array_equal(payload, np.arange(keys.size, dtype=np.int32))

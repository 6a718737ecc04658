"""File/CLI path (reference cli.py `sort` / `verify`, datagen.py read/write
formats): format round trips and exit codes on CPU; the GPU sort and device
verifier end to end against the oracle."""

import numpy as np
import pytest

from paper_2605_14419_b200 import cli


def test_bin_and_txt_round_trip(tmp_path):
    keys = np.random.default_rng(3).integers(-(2**63), 2**63 - 1, size=1001, dtype=np.int64, endpoint=True)
    for suffix in (".bin", ".txt"):
        p = tmp_path / f"k{suffix}"
        cli.write_keys(p, keys)
        np.testing.assert_array_equal(cli.read_keys(p), keys)
    # .bin is little-endian int64, byte for byte (datagen.py:187-188)
    assert (tmp_path / "k.bin").read_bytes() == keys.astype("<i8").tobytes()


def test_pinned_read_matches(tmp_path):
    torch = pytest.importorskip("torch")
    keys = np.arange(-50, 50, dtype=np.int64) * 7919
    p = tmp_path / "k.bin"
    cli.write_keys(p, keys)
    try:
        t = cli.read_keys(p, pinned=True)
    except RuntimeError:  # no pinned memory without a driver
        pytest.skip("pinned host memory needs a CUDA driver")
    np.testing.assert_array_equal(t.numpy(), keys)


def test_usage_and_corrupt_inputs(tmp_path):
    assert cli.main([]) == cli.USAGE_ERROR
    assert cli.main(["sort", "--in", "x.bin"]) == cli.USAGE_ERROR  # --out missing
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\x00" * 12)  # not a multiple of 8 bytes
    with pytest.raises(ValueError):
        cli.read_keys(bad)
    with pytest.raises(ValueError):
        cli.read_keys(tmp_path / "k.csv")
    with pytest.raises(ValueError):
        cli.write_keys(tmp_path / "k.csv", np.zeros(3, np.int64))


@pytest.mark.gpu
def test_sort_and_verify_files(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    keys = rng.integers(0, 5000, size=300_000, dtype=np.int64) * (1 << 40) - (1 << 60)
    src, out, perm = tmp_path / "in.bin", tmp_path / "out.bin", tmp_path / "perm.bin"
    cli.write_keys(src, keys)
    assert cli.main(["sort", "--in", str(src), "--out", str(out), "--perm", str(perm), "--stats"]) == 0
    ek, ep, _ = O.stable_sort(keys, np.arange(keys.size, dtype=np.int64))
    np.testing.assert_array_equal(cli.read_keys(out), ek)
    np.testing.assert_array_equal(cli.read_keys(perm), ep)
    assert cli.main(["verify", "--in", str(src), "--sorted", str(out), "--perm", str(perm)]) == 0
    assert cli.main(["verify", "--in", str(src), "--sorted", str(out)]) == 0
    # a broken permutation (two swapped equal keys) is caught: stability violation
    p = cli.read_keys(perm)
    j = int(np.flatnonzero(ek[1:] == ek[:-1])[0])
    p[[j, j + 1]] = p[[j + 1, j]]
    cli.write_keys(perm, p)
    assert cli.main(["verify", "--in", str(src), "--sorted", str(out), "--perm", str(perm)]) == cli.VERIFY_ERROR

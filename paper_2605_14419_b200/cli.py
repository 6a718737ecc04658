"""Command-line file path of the sort: ``sort`` and ``verify``.

Mirrors the reference CLI's ``zsort sort`` / ``zsort verify`` workflows
(/root/reference/pkg/src/zsort/cli.py:92-140, argument names and exit codes
from cli.py:1-30 and its parser) over the reference key-file format
(datagen.py:182-213: ``.bin`` = little-endian int64, ``.txt`` = one decimal
integer per line).  The sort runs on the GPU through the package's ``zsort``;
``.bin`` inputs are read straight into pinned host memory so the host->device
copy is a single DMA.  ``verify`` is the device structural checker (K8) in
place of the reference's numpy ``check_stable_permutation`` (verify.py:55-108).

Exit codes: 0 success, 1 verification failure, 2 usage errors and
unreadable or corrupt inputs (cli.py conventions).  The reference's ``gen``,
``bench``, ``alpha-sweep`` and ``report`` commands are harness and
presentation code around the path and are not rebuilt.

    python -m paper_2605_14419_b200 sort --in keys.bin --out sorted.bin --perm perm.bin --stats
    python -m paper_2605_14419_b200 verify --in keys.bin --sorted sorted.bin --perm perm.bin
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

USAGE_ERROR = 2
VERIFY_ERROR = 1


def read_keys(path, pinned: bool = False):
    """Read a key file (format by extension, datagen.py:197-213).  With
    ``pinned`` a ``.bin`` file lands directly in a pinned torch tensor."""
    p = Path(path)
    if p.suffix == ".bin":
        nbytes = os.path.getsize(p)
        if nbytes % 8 != 0:
            raise ValueError(f"{p}: size {nbytes} is not a multiple of 8 bytes")
        if pinned:
            import torch

            t = torch.empty(nbytes // 8, dtype=torch.int64, pin_memory=True)
            if nbytes:
                with open(p, "rb", buffering=0) as fh:
                    view = memoryview(t.numpy()).cast("B")
                    got = 0
                    while got < nbytes:
                        r = fh.readinto(view[got:])
                        if not r:
                            raise ValueError(f"{p}: short read")
                        got += r
            if sys.byteorder != "little":
                t = torch.from_numpy(t.numpy().byteswap())
            return t
        return np.fromfile(p, dtype="<i8").astype(np.int64)
    if p.suffix == ".txt":
        values = []
        with open(p) as fh:
            for line in fh:
                line = line.strip()
                if line:
                    values.append(int(line))
        arr = np.array(values, dtype=np.int64)
        if pinned:
            import torch

            return torch.from_numpy(arr).pin_memory()
        return arr
    raise ValueError(f"unsupported key file extension {p.suffix!r}; use .bin or .txt")


def write_keys(path, keys) -> None:
    """Write keys (datagen.py:182-194): ``.bin`` little-endian int64, ``.txt``
    one decimal integer per line."""
    p = Path(path)
    if p.suffix not in (".bin", ".txt"):
        raise ValueError(f"unsupported key file extension {p.suffix!r}; use .bin or .txt")
    if hasattr(keys, "numpy"):
        keys = keys.cpu().numpy()
    arr = np.ascontiguousarray(np.asarray(keys), dtype=np.int64)
    if p.suffix == ".bin":
        arr.astype("<i8").tofile(p)
    else:
        with open(p, "w") as fh:
            for v in arr.tolist():
                fh.write(f"{v}\n")


def cmd_sort(args) -> int:
    import torch

    from .core import SortConfig, zsort

    keys = read_keys(args.infile, pinned=True)
    n = keys.numel()
    payload = torch.arange(n, dtype=torch.int64).pin_memory()
    out = (torch.empty_like(keys).pin_memory(), torch.empty_like(payload).pin_memory())
    out_keys, out_payload, stats = zsort(keys, payload, SortConfig(alpha=args.alpha), out=out)
    if args.stats:
        print(f"zsort n={n} max_depth={stats.max_depth_reached} scatters={stats.total_scatter_passes} "
              f"counting={stats.counting_sort_invocations} insertion={stats.insertion_sort_invocations} "
              f"fallbacks={stats.fallback_invocations}", file=sys.stderr)
    write_keys(args.out, out_keys)
    if args.perm is not None:
        write_keys(args.perm, out_payload)
    return 0


def cmd_verify(args) -> int:
    import torch

    from .core import check_stable_permutation_device

    if not torch.cuda.is_available():
        raise RuntimeError("verify runs the device checker (K8) and needs a CUDA device")
    original = read_keys(args.infile, pinned=True)
    candidate = read_keys(args.sorted, pinned=True)
    if candidate.numel() != original.numel():
        print("verify: sorted file length mismatch", file=sys.stderr)
        return VERIFY_ERROR
    dev = torch.device("cuda", torch.cuda.current_device())
    d_in, d_out = original.to(dev), candidate.to(dev)
    if args.perm is not None:
        perm = read_keys(args.perm, pinned=True)
        if perm.numel() != candidate.numel():
            print("verify: permutation file length mismatch", file=sys.stderr)
            return VERIFY_ERROR
        viol = check_stable_permutation_device(d_in, d_out, perm.to(dev))
        print(f"stable_permutation violations={viol}", file=sys.stderr)
        return 0 if viol == 0 else VERIFY_ERROR
    # keys only: sorted, and a permutation of the input (compare with the
    # device sort of the input: a sorted permutation is unique)
    from .core import zsort

    ref, _, _ = zsort(d_in)
    ok_sorted = bool((d_out[1:] >= d_out[:-1]).all().item()) if d_out.numel() > 1 else True
    ok_perm = bool(torch.equal(ref, d_out))
    print(f"sorted={ok_sorted} permutation={ok_perm}", file=sys.stderr)
    return 0 if (ok_sorted and ok_perm) else VERIFY_ERROR


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="python -m paper_2605_14419_b200",
                                     description="B200 zSort: sort and verify key files")
    sub = parser.add_subparsers(dest="cmd", required=True)
    p_sort = sub.add_parser("sort", help="sort a key file")
    p_sort.add_argument("--in", dest="infile", required=True)
    p_sort.add_argument("--out", required=True)
    p_sort.add_argument("--algo", choices=["zsort"], default="zsort")
    p_sort.add_argument("--alpha", type=float, default=0.6)
    p_sort.add_argument("--stats", action="store_true", help="print SortStats to stderr")
    p_sort.add_argument("--perm", default=None, help="also write the stable permutation (original indices)")
    p_sort.set_defaults(func=cmd_sort)
    p_verify = sub.add_parser("verify", help="verify a sorted file against its original")
    p_verify.add_argument("--in", dest="infile", required=True)
    p_verify.add_argument("--sorted", required=True)
    p_verify.add_argument("--perm", default=None, help="permutation file written by sort --perm")
    p_verify.set_defaults(func=cmd_verify)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:  # argparse usage errors
        return USAGE_ERROR if exc.code else 0
    try:
        return args.func(args)
    except (OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return USAGE_ERROR


if __name__ == "__main__":
    sys.exit(main())

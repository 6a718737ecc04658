import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_14419_b200 as Z
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**8
mapping = sys.argv[2] if len(sys.argv) > 2 else "fitted"
keys, pay = O.make_config(4, n)
tk = torch.from_numpy(keys).cuda()
tp = torch.arange(n, dtype=torch.int64, device="cuda")
k, p, st = Z.zsort(tk, tp, Z.SortConfig(mapping=mapping))
print("stats", st, flush=True)
print("device violations", Z.check_stable_permutation_device(tk, k, p))
ok = k.cpu().numpy(); op = p.cpu().numpy()
o = O.ordered_u64(ok)
bad_sorted = np.flatnonzero(o[1:] < o[:-1])
print("unsorted positions", bad_sorted.size, bad_sorted[:10])
eq = o[1:] == o[:-1]
bad_stable = np.flatnonzero(eq & (op[1:] <= op[:-1]))
print("unstable positions", bad_stable.size, bad_stable[:10])
perm_ok = np.array_equal(np.sort(op), np.arange(n))
print("permutation", perm_ok)
print("key match", np.array_equal(ok.view(np.uint64), keys[op].view(np.uint64)) if perm_ok else "n/a")
for j in list(bad_sorted[:3]) + list(bad_stable[:3]):
    lo, hi = max(0, j - 3), min(n, j + 5)
    print(j, ok[lo:hi], op[lo:hi])

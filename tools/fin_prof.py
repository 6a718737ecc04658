import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_14419_b200 as Z
from oracle import oracle as O
keys, pay = O.make_config(2)
tk = torch.from_numpy(keys).cuda(); tp = torch.from_numpy(pay).cuda()
for _ in range(2): Z.zsort(tk, tp)
torch.cuda.synchronize()
os.environ["ZSB_FIN_PROFILE"] = "1"
Z.zsort(tk, tp)

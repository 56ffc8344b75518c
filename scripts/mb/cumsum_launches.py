import sys; sys.path.insert(0, '.')
import torch, paper_2109_13504_b200 as mg
from oracle import oracle
import os
w = torch.from_numpy(oracle.gen_gaussian_weights(4.0, 1 << 24, 31337, os.environ.get("PREC", "single"))).cuda()
for _ in range(3):
    c = mg.inclusive_prefix(w)
torch.cuda.synchronize()

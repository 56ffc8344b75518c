"""Resolver profile of the exact cumsum at 2^24 (needs a -DMGP_PX_PROF build of libmgp.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2109_13504_b200 as mg
from paper_2109_13504_b200 import _lib
from oracle import oracle
names = ["super_windows", "super_cyc", "chunk_windows", "chunk_cyc", "crossing_chunks", "crossing_cyc",
         "block_passes", "seq_tails", "seq_elems", "kernel_cyc", "load_cyc", "pass_cyc", "tail_cyc", "tail0_c*4096+p", "tail1", "tail2"]
for prec in ("single", "double"):
    w = torch.from_numpy(oracle.gen_gaussian_weights(4.0, 1 << 24, 31337, prec)).cuda()
    mg.inclusive_prefix(w); torch.cuda.synchronize()
    buf = (ctypes.c_int64 * 16)()
    _lib.check(_lib.lib().mgp_debug_px_prof(buf, 1))
    mg.inclusive_prefix(w); torch.cuda.synchronize()
    _lib.check(_lib.lib().mgp_debug_px_prof(buf, 1))
    print(prec, {k: int(v) for k, v in zip(names, buf[:16])})

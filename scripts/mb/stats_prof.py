"""ncu target: the B-rule statistics (mgp_weight_stats) on 2^24 float32 weights."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2109_13504_b200 as mg  # noqa: E402
from paper_2109_13504_b200 import _device as D  # noqa: E402
from paper_2109_13504_b200 import _lib  # noqa: E402

wv = mg.gen_gaussian_weights(mg.GaussianWeightParams(4.0, 1 << 24), 7, "single", device="cuda")
out = torch.empty(16, dtype=torch.float64, device="cuda")
for _ in range(3):
    _lib.check(_lib.lib().mgp_weight_stats(D.ptr(wv.values), 0, 1 << 24, D.ptr(out), D.stream_ptr()))
torch.cuda.synchronize()

"""Config-5 forward + dL/da probe (for ncu captures of the batch kernels)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_20870_b200 as fg  # noqa: E402
import prep  # noqa: E402

fs, orders, feats, l = prep.config5()
G, n, C = feats.shape
batch = fg.GraphBatch(fs, l)
a = torch.from_numpy(orders).cuda()
x = torch.from_numpy(np.ascontiguousarray(feats.transpose(0, 2, 1)).astype(np.complex64)).cuda()
g = torch.randn((G, orders.shape[1], C, n), dtype=torch.complex64, device="cuda")
for _ in range(3):
    batch.forward(a, x)
    batch.dlda(a, g, x)
torch.cuda.synchronize()
print("c5 probe ok")

"""One device-resident launch of one fixed-width or varlen batch (for an
`ncu --set full --import-source on` capture of that kernel).

usage: python tools/ncu_one.py md5 65536 1024      (fixed)
       python tools/ncu_one.py md5 varlen           (configs[3] batch)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

alg = sys.argv[1]
if sys.argv[2] == "varlen":
    n = 1 << 22
    lens = np.random.default_rng(4).integers(1, 4097, n).astype(np.int64)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    data = torch.empty(int(off[-1]), dtype=torch.uint8, device="cuda:0")
    device.fill_random(data, 4)
    d_off = torch.from_numpy(off).cuda()
    for _ in range(2):
        device.hash_varlen(alg, data, d_off, offset_base=0)
else:
    n, L = int(sys.argv[2]), int(sys.argv[3])
    buf = torch.empty(n * L, dtype=torch.uint8, device="cuda:0")
    device.fill_random(buf, 2)
    for _ in range(2):
        device.hash_fixed(alg, buf.view(n, L))
torch.cuda.synchronize()
print(_native.last_kernel_name())

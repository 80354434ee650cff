"""k_histogram_u8 on the C3 image (16.7 MB bimodal u8), CUDA events; not a bench value."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2510_14982_b200 import imaging

rnd = np.random.default_rng(0)
n = 4096 * 4096
comp = rnd.random(n) < 0.5
img = np.clip(np.rint(np.where(comp, rnd.normal(70.0, 12.0, n), rnd.normal(190.0, 14.0, n))), 0, 255).astype(np.uint8)
d = torch.as_tensor(img).cuda()
c = imaging.histogram_device(d)
assert np.array_equal(c.cpu().numpy(), np.bincount(img, minlength=256)), "histogram differs from bincount"
for extra in (1, 15, 4096 * 4096 * 3 + 7):  # ragged tail; > 65520 pixels per thread (early folds)
    x = torch.as_tensor(rnd.integers(0, 256, extra, dtype=np.uint8)).cuda()
    assert np.array_equal(imaging.histogram_device(x).cpu().numpy(), np.bincount(x.cpu().numpy(), minlength=256))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    imaging.histogram_device(d)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 50 * 1e3
print(f"k_histogram_u8: {us:.1f} us for {n / 1e6:.1f} MB = {n / us / 1e3:.0f} GB/s")

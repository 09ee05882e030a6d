"""DMMA pipe throughput vs accumulator chains per warp and operand source
(registers vs a shared-memory load per DMMA), 16 warps per SM."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_17626_b200 import _lib  # noqa: E402

L = _lib.lib()
out = torch.zeros(4, dtype=torch.float64, device="cuda")
grid, iters = 148, 20000
for mode in (1, 11, 12, 14, 18, 21, 22, 24, 28):
    ch = mode % 10 if mode > 1 else 4
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = L.fl_probe_fp64(mode, grid if mode > 1 else 296, iters, C.c_void_p(out.data_ptr()), None)
        e1.record()
        torch.cuda.synchronize()
    assert rc == 0, rc
    ms = e0.elapsed_time(e1)
    warps = grid * 16 if mode > 1 else 296 * 8
    fl = warps * iters * ch * 512
    print(f"mode {mode:2d} chains {ch} {'lds' if mode > 20 else 'reg'}: {fl / ms / 1e9:.2f} TF/s")

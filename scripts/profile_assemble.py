"""Two K1 launches of a config's assembly (the second is the one to profile):

    ncu --set full -k regex:assemble_kernel -s 1 -c 1 -o gpurun_out/asm python scripts/profile_assemble.py cfg4
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_17626_b200 import workloads  # noqa: E402
from paper_2506_17626_b200.assembly import AssemblyPlan  # noqa: E402

if __name__ == "__main__":
    wl = workloads.build(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
    plan = AssemblyPlan(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
    store = plan.new_store()
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch(store)
        e1.record()
        torch.cuda.synchronize()
        print(f"K1 {e0.elapsed_time(e1):.3f} ms", flush=True)

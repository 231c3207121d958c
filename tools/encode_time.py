"""Time the GPU E8P encoder on a 70B-MLP-sized matrix (28672 x 8192 -> 29.4 M 8-vectors)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2402_04396_b200 as q8p
v = torch.randn(28672 * 8192 // 8, 8, dtype=torch.float64, device="cuda")
q8p.e8p_encode(v[:1000])
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); w = q8p.e8p_encode(v); b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b)
print(f"e8p_encode 28672x8192 ({v.shape[0]} blocks): {ms:.1f} ms  ({v.shape[0] / ms / 1e3:.1f} M blocks/s)")

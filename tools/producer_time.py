"""GPU producer timing at the 70B MLP shape (H = I route): W~ = T_u W T_v^T in f64
(q8p_rht_cols_f64, both sides) + 2-bit RVQ codes (q8p_rvq_quantize).  Synthetic W."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2402_04396_b200 as q8p
m, n = 28672, 8192
w = torch.randn(m, n, dtype=torch.float64, device="cuda")
su = torch.randint(0, 256, ((m + 7) // 8,), dtype=torch.uint8, device="cuda")
sv = torch.randint(0, 256, ((n + 7) // 8,), dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
q8p.rht_cols_f64(w, su)
wt = w.t().contiguous()
q8p.rht_cols_f64(wt, sv)
w2 = wt.t().contiguous()
torch.cuda.synchronize()
t1 = time.perf_counter()
codes = q8p.rvq_quantize(w2.view(-1, 8), [(q8p.CB_E8P_2BIT, 1.11)])
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"28672x8192 producer on GPU: transforms {1e3 * (t1 - t0):.1f} ms, E8P codes {1e3 * (t2 - t1):.1f} ms")

import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2502_03000_b200.batch import atb_schur_trace
bt, n = 20000, 128
ops = [torch.rand((bt, n, n), dtype=torch.float32, device="cuda").transpose(1, 2) for _ in range(4)]
E, s = atb_schur_trace(*ops)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); E, s = atb_schur_trace(*ops); e1.record(); torch.cuda.synchronize()
print("ms", e0.elapsed_time(e1), "per instance per CTA us", e0.elapsed_time(e1) * 1e3 / (bt / 296))

import sys, json, torch
sys.path.insert(0, "/root/repo")
import paper_2007_06289_b200 as pkg, phantoms as P
c = json.load(open("/root/repo/coeffs/iir_q3_n64_dc0.json"))
for B in (1, 64, 4096):
    plan = pkg.Plan(64, c["b"], c["a"], max_batch=B)
    S = P.random_linogram(64, B, seed=1).cuda()
    out = torch.empty((B, 64, 64), device="cuda")
    for _ in range(3): plan.reconstruct(S, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): plan.reconstruct(S, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"N=64 B={B}: {ms:.4f} ms per call, {B/ms*1e3:.0f} slices/s, path frac {B*36*64*64/(ms*1e-3)/6458.1e9:.3f}", flush=True)

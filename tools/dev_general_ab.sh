# A/B of the general-path pass A launch bound (run under gpurun): config-1 and N=256 timing
set -e
cat > /tmp/gen_t.py <<'PY'
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2007_06289_b200 as pkg, phantoms as P
for N, B in ((64, 4096), (256, 256), (8192, 1)):
    c = json.load(open(f"coeffs/iir_q3_n{min(N,4096)}_dc0.json"))
    plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
    S = P.random_linogram(N, 1, seed=1).cuda().expand(B, -1, -1, -1).contiguous()
    img = torch.empty((B, N, N), device="cuda")
    for _ in range(3): plan.reconstruct(S, out=img)
    torch.cuda.synchronize(); plan.profile(True)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for _ in range(10): plan.reconstruct(S, out=img)
    e1.record(); torch.cuda.synchronize(); kt = plan.kernel_times(); plan.profile(False)
    print("N", N, "B", B, "ms/call", round(e0.elapsed_time(e1) / 10, 4), {k: round(v[0] / 10, 4) for k, v in kt.items() if v[1]})
    del S, img, plan; torch.cuda.empty_cache()
PY
python -m paper_2007_06289_b200.build >/dev/null; echo "bound (256,1):"; python /tmp/gen_t.py
sed -i 's/__launch_bounds__(kThreads, 1) k_fht_a(/__launch_bounds__(kThreads, 2) k_fht_a(/' paper_2007_06289_b200/csrc/fht.cu
python -m paper_2007_06289_b200.build >/dev/null; echo "bound (256,2):"; python /tmp/gen_t.py

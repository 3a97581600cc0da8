"""Developer: forward FHT at several N, exact vs the oracle on integer images."""
import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg
import phantoms as P
from oracle import fbp_oracle as O
for N in [int(a) for a in sys.argv[1:]]:
    c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{min(max(N, 64), 4096)}_dc0.json")))
    plan = pkg.Plan(N, c["b"], c["a"], max_batch=1)
    img = P.integer_image(N, 1, seed=1, lo=-7, hi=7)
    try:
        out = plan.forward(img.cuda()).cpu().numpy()[0]
        torch.cuda.synchronize()
    except Exception as e:
        print(N, "ERR", str(e)[:200]); break
    ref = O.fht_forward(img[0].numpy().astype(np.float64))
    bad = np.argwhere(out != ref)
    print(N, "mismatch", len(bad), bad[:5].tolist(), flush=True)

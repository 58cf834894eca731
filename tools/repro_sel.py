import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19449_b200 as rsp
x = np.fromfile(os.path.join(os.path.dirname(os.path.abspath(__file__)), "x_sign_dups.bin"), dtype=np.float32)
xt = torch.from_numpy(x).cuda()
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    kept, rest = rsp.top_k_by_magnitude(xt, 31, with_rest=True)
    got = kept.cpu().numpy()
    if 3840 not in got or 493 in got:
        bad += 1
print("bad", bad)

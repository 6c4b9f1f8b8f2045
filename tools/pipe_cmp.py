import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2602_12242_b200 as mx
from oracle import magnex_oracle as O
def build(g, pipe):
    os.environ["MXB_PIPE"] = pipe
    return mx.DemagKernel.build(g, symmetric=True)
for dims in [(16, 512, 512), (64, 512, 512)] if len(sys.argv) < 2 else [tuple(int(v) for v in sys.argv[1:4])]:
    g = mx.GridSpec(*dims, 2e-9, 2.5e-9, 3e-9)
    m = np.random.default_rng(1).normal(size=(3,) + g.shape) * 8e5
    h5 = build(g, "0").field(m)
    hw = build(g, "1").field(m)
    print(dims, "rel diff warp-pipe vs 5-pass:", np.linalg.norm(hw - h5) / np.linalg.norm(h5), "max", np.max(np.abs(hw-h5))/np.max(np.abs(h5)), flush=True)

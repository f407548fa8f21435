import sys, re
sys.path.insert(0, '.')
import numpy as np
import paper_1712_05878_b200 as g
from oracle import oracle as O
ctx = g.Context(0)
for arch_text in ["lstm(7,33,3),dense(33,17,tanh),dense(17,9,identity),softmax(9,5)", "lstm(5,8,10),dense(8,64,relu),dense(64,48,tanh),softmax(48,3)", "lstm(10,50,20),dense(50,32,relu),softmax(32,4)"]:
  for n in (1, 37):
    arch = g.Architecture(ctx, arch_text)
    D, H, T = map(int, re.match(r"lstm\((\d+),(\d+),(\d+)\)", arch_text).groups())
    K = g.arch_info(arch_text)[2]
    x, y = g.generate(g.data_spec(1, n, seq_len=T, input_dim=D, n_classes=K, delta=1.0, seed=1234))
    w = g.init_weights(arch, 7).astype(np.float32)
    gg, lo = g.forward_backward(w, arch, x, y)
    go, _, loo = O.forward_backward(O.parse_arch(arch_text), w.astype(np.float64), x.astype(np.float64), y)
    print(arch_text, n, arch.kernel_name, "loss", lo, loo)
    for (off, d0, d1) in arch.tensors():
        m = d0*max(d1,1); a = gg[off:off+m]; b = go[off:off+m]
        print("  ", off, d0, d1, np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-30), np.abs(b).max())

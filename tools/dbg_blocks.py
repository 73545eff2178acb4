import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from paper_2004_11610_b200 import inputs as I, xc
N, B, eps = 512, 1, 1e-12
kind = O.Kind(O.KIND_JACOBI, 0.0, 0.0)
x, _, _ = O.gauss_rule(kind, N)
X = I.rhs(N, B, 100)
T = xc.Transform(xc.XC_JACOBI, x, eps)
Y = T.apply(torch.from_numpy(X).cuda()).cpu().numpy()
op = O.compress(O.make_plan(kind, N, eps), x)
Ya = O.apply_output_axis(op, X)
info = T.info(); print(info['n_blocks'], info['tail'])
for i in range(info['n_blocks']):
    b = T.block_info(i); lo, hi = b['m_off'] + b['keep_lo'], b['m_off'] + b['keep_hi']
    print(i, b, 'err', np.abs(Y[lo:hi] - Ya[lo:hi]).max(), 'scale', np.abs(Ya[lo:hi]).max())
t = info['tail']; print('tail err', np.abs(Y[:t] - Ya[:t]).max())

import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2411_16127_b200 import fused
dev = torch.device('cuda')
for K, M, N in [(33, 8, 16), (32, 128, 16), (64, 128, 16), (1024, 64, 64), (1056, 64, 64), (2048, 64, 64), (50000, 64, 64)]:
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (K, M)).astype(np.float32); dY = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ref = X.T.astype(np.float64) @ dY.astype(np.float64)
    C = fused.gemm(torch.from_numpy(X).to(dev), torch.from_numpy(dY).to(dev), trans_a=True).cpu().numpy()
    err = np.abs(C - ref).max() / max(1, np.abs(ref).max())
    print(K, M, N, 'err', err, 'zeros', (C == 0).mean(), 'C[0,:4]', C[0, :4], 'ref', ref[0, :4], flush=True)

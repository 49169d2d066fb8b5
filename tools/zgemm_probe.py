import torch, time
n=1050625
for m in (5, 25, 49):
    V=torch.randn(m, n, dtype=torch.complex128, device='cuda')   # columns contiguous (row-major m x n == col-major n x m)
    W=torch.randn(4, n, dtype=torch.complex128, device='cuda')
    for _ in range(3):
        C=V.conj() @ W.T        # m x 4  (V^H W)
        W2=W - (C.T @ V)        # 4 x n  (W - V C)^T
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        C=V.conj() @ W.T
    e1.record(); torch.cuda.synchronize(); t1=e0.elapsed_time(e1)/10
    e0.record()
    for _ in range(10):
        W2=torch.addmm(W.T, V.T, C, beta=1, alpha=-1)
    e1.record(); torch.cuda.synchronize(); t2=e0.elapsed_time(e1)/10
    print(f"m={m}: V^H W {t1*1e3:.0f} us ({m*n*16/t1/1e6:.0f} GB/s)  W - V C {t2*1e3:.0f} us ({m*n*16/t2/1e6:.0f} GB/s)")

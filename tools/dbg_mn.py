import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1907_05013_b200 import _lib
def run(M,N,K,amn,bmn,bn=64,splits=1):
    g=np.random.default_rng(0)
    A=g.standard_normal((M,K)).astype(np.float32); B=g.standard_normal((N,K)).astype(np.float32)
    dA=torch.from_numpy(np.ascontiguousarray(A.T if amn else A)).cuda(); dB=torch.from_numpy(np.ascontiguousarray(B.T if bmn else B)).cuda()
    dD=torch.zeros((splits,M,N),device='cuda')
    st=_lib.lib.pooch_op_gemm_test(C.c_void_p(dA.data_ptr()),C.c_void_p(dB.data_ptr()),C.c_void_p(dD.data_ptr()),M,N,K,amn,bmn,bn,splits,None)
    torch.cuda.synchronize()
    D=dD.cpu().numpy().astype(np.float64).sum(0); ref=A.astype(np.float64)@B.astype(np.float64).T
    return st, float(np.linalg.norm(D-ref)/np.linalg.norm(ref)), float(np.abs(D).max())
for amn,bmn in [(1,0),(2,0),(0,1),(0,2),(1,1),(2,2)]:
    for (M,N,K) in [(128,64,32),(128,64,64),(256,128,96)]:
        print(amn,bmn,M,N,K, run(M,N,K,amn,bmn))

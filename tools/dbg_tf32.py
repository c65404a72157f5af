import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1907_05013_b200 import _lib
def trunc(a):
    return (a.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
def rn(a):
    u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x1000) & 0xFFFFE000  # round half up on magnitude bits
    return u.astype(np.uint32).view(np.float32)
def rne(a):
    u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 13) & 1
    u = (u + 0xFFF + lsb) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)
M,N,K=512,256,1024
g=np.random.default_rng(0)
A=g.standard_normal((M,K)).astype(np.float32); B=g.standard_normal((N,K)).astype(np.float32)
dA=torch.from_numpy(A).cuda(); dB=torch.from_numpy(B).cuda(); dD=torch.zeros((M,N),device='cuda')
_lib.lib.pooch_op_gemm_test(C.c_void_p(dA.data_ptr()),C.c_void_p(dB.data_ptr()),C.c_void_p(dD.data_ptr()),M,N,K,0,0,256,1,None)
torch.cuda.synchronize(); D=dD.cpu().numpy().astype(np.float64)
for nm,f in [('exact',lambda a:a),('trunc',trunc),('rn',rn),('rne',rne)]:
    ref=f(A).astype(np.float64)@f(B).astype(np.float64).T
    print(nm, np.linalg.norm(D-ref)/np.linalg.norm(ref), np.abs(D-ref).max())

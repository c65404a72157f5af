import ctypes as C, numpy as np, torch, sys, os
sys.path.insert(0, '.')
from paper_1907_05013_b200 import _lib
from oracle import layers as L
def run(N,H,W,Cin,K,R,s,p):
    g=np.random.default_rng(1)
    x=g.standard_normal((N,H,W,Cin)).astype(np.float32); ho,wo=L.conv_out_hw(H,W,R,R,s,p)
    gy=g.standard_normal((N,ho,wo,K)).astype(np.float32)
    d=_lib.ConvDesc(N,H,W,Cin,K,R,R,s,p)
    wsb=_lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
    ws=torch.empty(max(wsb//4,1),device='cuda'); ddw=torch.full((K,R,R,Cin),float('nan'),device='cuda')
    dx=torch.from_numpy(x).cuda(); dg=torch.from_numpy(gy).cuda()
    st=_lib.lib.pooch_op_conv_wgrad(C.byref(d),C.c_void_p(dx.data_ptr()),C.c_void_p(dg.data_ptr()),C.c_void_p(ddw.data_ptr()),C.c_void_p(ws.data_ptr()),wsb,None)
    torch.cuda.synchronize()
    ref=L.conv2d_wgrad(x.transpose(0,3,1,2).astype(np.float64),gy.transpose(0,3,1,2).astype(np.float64),(K,Cin,R,R),s,p).transpose(0,2,3,1)
    r=np.linalg.norm(ddw.cpu().numpy()-ref)/np.linalg.norm(ref)
    return st, wsb, float(r)
cases=[(16,56,56,64,64,3,1,1),(2,56,56,64,64,3,1,1),(16,14,14,64,64,3,1,1),(16,56,56,32,32,3,1,1),(4,56,56,64,64,1,1,0),(16,28,28,64,64,3,1,1),(8,56,56,64,64,3,1,1)]
for sp in [None,'1','2','8']:
    if sp: os.environ['POOCH_WGRAD_SPLITS']=sp
    for c in cases: print(sp, c, run(*c), flush=True)

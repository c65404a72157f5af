import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1907_05013_b200 import _lib
M,N,K=128,64,32
g=np.random.default_rng(0)
A=g.standard_normal((M,K)).astype(np.float32); B=g.standard_normal((N,K)).astype(np.float32)
for amn,bmn in [(0,0),(1,0),(0,1),(2,0),(0,2),(1,1)]:
    dA=torch.from_numpy(np.ascontiguousarray(A.T if amn else A)).cuda(); dB=torch.from_numpy(np.ascontiguousarray(B.T if bmn else B)).cuda()
    stage=(128*32+64*32)
    dD=torch.zeros(M*N+stage,device='cuda')
    st=_lib.lib.pooch_op_gemm_test(C.c_void_p(dA.data_ptr()),C.c_void_p(dB.data_ptr()),C.c_void_p(dD.data_ptr()),M,N,K,amn,bmn,64,101,None)
    torch.cuda.synchronize()
    out=dD.cpu().numpy(); D=out[:M*N].reshape(M,N); sm=out[M*N:]
    smA=sm[:128*32]; smB=sm[128*32:]
    # expected K-major: chunk(row,j) at ((j*(R/8)+row/8)*128+(row%8)*16)/4 floats
    def kmaj(X,R):
        e=np.zeros(R*32,np.float32)
        for r in range(R):
            for j in range(8):
                o=((j*(R//8)+r//8)*128+(r%8)*16)//4
                e[o:o+4]=X[r,4*j:4*j+4]
        return e
    def mnmaj(X,R):  # X [R][K]
        e=np.zeros(R*32,np.float32)
        for gq in range(R//4):
            for k in range(32):
                r=k%8; c=gq%8
                o=((((k//8)*(R//32)+gq//8)*1024)+r*128+((c^r)*16))//4
                e[o:o+4]=X[4*gq:4*gq+4,k]
        return e
    eA=mnmaj(A,128) if amn else kmaj(A,128)
    amn_=amn
    eB=mnmaj(B,64) if bmn else kmaj(B,64)
    ref=A.astype(np.float64)@B.astype(np.float64).T
    print(amn,bmn,'st',st,'smA ok',np.array_equal(smA,eA),'smB ok',np.array_equal(smB,eB),'D rel',np.linalg.norm(D-ref)/np.linalg.norm(ref), 'nnzA', np.count_nonzero(smA), 'nnzB', np.count_nonzero(smB))
exec(open('tools/dbg_mn.py').read().split('for amn,bmn')[0])
for amn,bmn in [(1,0),(0,1),(1,1)]:
    for (M,N,K) in [(128,64,32),(256,128,96),(384,256,520)]:
        for bn in (64,128,256):
            print(amn,bmn,M,N,K,bn, run(M,N,K,amn,bmn,bn))

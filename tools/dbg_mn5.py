import ctypes as C
exec(open('tools/dbg_mn.py').read().split('for amn,bmn')[0])
L=_lib.lib
L.pooch_dbg_set.argtypes=[C.c_int]*5
res=[]
# smem layout is SW128 MN-major: atoms 1024B, mn-atom stride 1024, k-group stride 4096 (M=128)
for layout in (0,1,2,4,6):
  for lbo in (16, 128, 1024, 4096):
    for sbo in (16, 128, 1024, 4096):
      for step in (4096, 1024):
        for ix in (0, 1<<15):
          L.pooch_dbg_set(lbo,sbo,layout,step,ix)
          st,r,mx=run(128,64,32,1,0)
          if mx != 0.0:
              res.append((layout,lbo,sbo,step,ix,r,mx)); print(res[-1], flush=True)
L.pooch_dbg_set(0,0,0,0,0)
# also idesc xor of the transpose bit only (A loaded MN-major but flagged K-major)
L.pooch_dbg_set(0,0,0,0,1<<15)
print('xor15 with MN data', run(128,64,32,1,0))
L.pooch_dbg_set(0,0,0,0,0)
print('done', len(res))

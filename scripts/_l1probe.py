import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, time
from paper_1711_05017_b200 import backend as be
from conftest import synthetic_window, random_rotation
rng=np.random.default_rng(0)
w=64
W1,W2=be.DeviceWindow(synthetic_window(rng,w)),be.DeviceWindow(synthetic_window(rng,w))
n=2000
Rs=np.stack([random_rotation(rng) for _ in range(n)]); ts=rng.uniform(-1,1,(n,3))
R0=Rs[0]; t0=ts[0]
def jit(i):
    a=0.5*np.pi/180*np.sin(i*0.01)
    c,s=np.cos(a),np.sin(a)
    return R0@np.array([[c,-s,0],[s,c,0],[0,0,1.0]]), t0+0.001*np.sin(i*0.02)
cases={"random":[(Rs[i],ts[i]) for i in range(n)], "same":[(R0,t0)]*n, "jitter":[jit(i) for i in range(n)]}
with be.HapticServer(W1,W2,False,(0.1,)*3,1.0,(0.1,0.2,0.3)) as srv:
    for name,poses in cases.items():
        for R,t in poses[:200]: be.cascade(W1,W2,False,(0.1,)*3,1.0,R,t,(0.1,0.2,0.3))
        g=[];h=[]
        for R,t in poses:
            t1=time.perf_counter(); be.cascade(W1,W2,False,(0.1,)*3,1.0,R,t,(0.1,0.2,0.3)); h.append(time.perf_counter()-t1); g.append(srv.last_timing()['gpu_us'])
        print(f"{name}: server gpu p50 {np.median(g):.2f} us  host p50 {1e6*np.median(h):.2f} us", flush=True)

python - << 'PY'
import sys, time
sys.path.insert(0,'.')
import numpy as np, graphgen as gg, paper_1602_00963_b200 as bcb
g = gg.rmat(20,16,seed=1); S = gg.sample_sources(g, 65536, seed=2)
G = bcb.Graph.from_csr(g); G.set_option(bcb.OPT_PROFILE,1)
for chunk in (8192, 16384, 65536):
    G.compute(S[:chunk])
    t=time.perf_counter(); tot=0
    for i in range(0, 65536, chunk):
        G.compute(S[i:i+chunk]); st=G.stats(); tot+=st['fwd_hits']
    dt=time.perf_counter()-t
    print(chunk, f"{dt:.3f}s", f"{65536*g.m/dt/1e9:.1f} GTEPS", "hits", tot)
PY

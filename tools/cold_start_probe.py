import time, sys, os
t0=time.perf_counter()
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
t1=time.perf_counter(); print("import torch", t1-t0)
import paper_2407_02740_b200 as vg
from paper_2407_02740_b200 import _cabi, engine
t2=time.perf_counter(); print("import pkg", t2-t1)
lib=_cabi.load(); t3=time.perf_counter(); print("load lib", t3-t2)
torch.cuda.init(); torch.zeros(1,device="cuda"); torch.cuda.synchronize(); t4=time.perf_counter(); print("cuda ctx via torch", t4-t3)
rng=np.random.default_rng(0); n=10000
locs=rng.uniform(size=(n,2)); y=rng.normal(size=n); X=np.ones((n,1))
nn=vg.find_ordered_neighbors(locs,30); t5=time.perf_counter(); print("neighbors", t5-t4)
prob=engine.DeviceProblem(vg.Dataset(y,X,locs),nn,"exponential_isotropic"); t6=time.perf_counter(); print("DeviceProblem", t6-t5)
prob.totals(np.array([1.0,0.1,0.1])); t7=time.perf_counter(); print("first eval", t7-t6)
prob.totals(np.array([1.0,0.1,0.1])); t8=time.perf_counter(); print("second eval", t8-t7)

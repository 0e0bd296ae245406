import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle, workloads as W
from paper_2510_15330_b200 import Simulator
w=W.config_c1()
w.scenarios[0].record |= 2; w.scenarios[1].record |= 2
cols=w.columns()
sim=Simulator(cols); sim.run(); torch.cuda.synchronize()
st=sim.stats()
rows,ctrl=sim.series(1)
o=oracle.run_scenario(cols,1,rows_cap=1000,ctrl_log_cap=1000)
oc=o['ctrl_log']
print("gpu",len(ctrl),"orc",len(oc), "active_ingests", st[1]['active_ingests'], o['active_ingests'])
for i in range(max(len(ctrl),len(oc))):
    g=tuple(int(x) for x in ctrl[i])[:5] if i<len(ctrl) else None
    e=(oc[i]['second'],oc[i]['sample'],oc[i]['k'],oc[i]['r_bp'],oc[i]['active']) if i<len(oc) else None
    flag = "" if g==e else "  <<<"
    print(i,g,e,flag)

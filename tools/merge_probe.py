import os,sys
os.environ["NX_PHASE_TIMERS"]="2"; os.environ["NX_SO"]="/root/repo/tools/_timers/_nxsched.so"
sys.path.insert(0,"/root/repo")
from paper_2509_23384_b200 import sim, workloads as W
cfgs=[W.sweep_replica(r,1,p,2000) for r in (10.0,47.5) for p in ("prism",)]
b=sim.Batch(cfgs); b.run()
for i,c in enumerate(cfgs):
    cy=b.phase_cycles(i); s=b.summaries()[i]
    print(c['workload']['rate'], "events",s.events,"merge_s",cy[0]/1.965e9,"calls",cy[12],"merged",cy[13],"empty",cy[14],"catchup_s",cy[15]/1.965e9)

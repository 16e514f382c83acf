import os, sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
os.environ["CACTO_CRITIC_TC_MIN"]="0"
import paper_2602_19699_b200 as P
P.set_precision("fp32")
from test_gpu_critic_tc import nets, batch
from paper_2602_19699_b200 import nets as B_nets, specs as B_specs
from oracle import nets as O_nets
for name in ("toy1d","dubins"):
    spec,_=B_specs.config(name); rng=np.random.default_rng(31)
    critic,target=nets(spec,rng); b=batch(spec,1000,rng)
    for boot in (False,True):
        loss,g=B_nets.critic_loss(critic,target,b,0.7,boot)
        ref,rg=O_nets.critic_loss(critic,target,b,0.7,boot)
        os.environ["CACTO_CRITIC_TC"]="0"
        ls,gs=B_nets.critic_loss(critic,target,b,0.7,boot)
        os.environ.pop("CACTO_CRITIC_TC")
        sc=max(np.abs(r).max() for r in rg)
        print(name, boot, "loss", loss, ref, ls)
        for i,(x,r,y) in enumerate(zip(g,rg,gs)):
            print("  p%d"%i, x.shape, "tc %.2e simt %.2e"%(np.abs(x-r).max()/sc, np.abs(y-r).max()/sc), "max|r| %.2e"%np.abs(r).max())

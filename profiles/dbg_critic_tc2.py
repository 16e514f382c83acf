import os, sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
os.environ["CACTO_CRITIC_TC_MIN"]="0"
import paper_2602_19699_b200 as P
P.set_precision("fp32")
from test_gpu_critic_tc import nets, batch
from paper_2602_19699_b200 import nets as B_nets, specs as B_specs
from oracle import nets as O_nets
spec,_=B_specs.config("toy1d"); rng=np.random.default_rng(31)
critic,target=nets(spec,rng)
for R in (128, 256, 1000):
    b=batch(spec,R,rng)
    for boot in (False, True):
        for ks in (0.0, 0.7):
            ref,_=O_nets.critic_loss(critic,target,b,ks,boot)
            vals=[B_nets.critic_loss(critic,target,b,ks,boot)[0] for _ in range(3)]
            print(R, boot, ks, "ref %.6f"%ref, " ".join("%.6f"%v for v in vals))

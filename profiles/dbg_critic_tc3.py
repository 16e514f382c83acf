import os, sys, ctypes, numpy as np, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
os.environ["CACTO_CRITIC_TC_MIN"]="0"
import paper_2602_19699_b200 as P
P.set_precision("fp32")
from test_gpu_critic_tc import nets, batch
from paper_2602_19699_b200 import nets as B_nets, specs as B_specs, _lib
from paper_2602_19699_b200.device import device_net
from paper_2602_19699_b200.nets import _Batch
from oracle import nets as O_nets
spec,_=B_specs.config("toy1d"); rng=np.random.default_rng(31)
critic,target=nets(spec,rng)
R=128
b=batch(spec,R,rng)
net=device_net(critic); bb=_Batch(b)
L=_lib.load(); nbytes=L.cacto_loss_workspace_bytes(net.desc, R)
P_=net.count
def al(x): return (x+255)&~255
off=al((P_+1)*4); offs={}
for l in range(3): offs['GZ%d'%l]=off; off+=al(2*R*64*4)
offs['UA0']=off; off+=al(2*R*16*4)
offs['UA1']=off; off+=al(2*R*64*4)
offs['UA2']=off; off+=al(2*R*64*4)
offs['U3']=off; off+=al(R*64*4)
offs['A3']=off; off+=al(R*64*4)
offs['DEL']=off
pre,acts,o=O_nets.forward_caches(critic,b.xa)
for trial in range(3):
    ws=torch.zeros(nbytes,dtype=torch.uint8,device='cuda'); npart=ctypes.c_int32(0)
    _lib.call("cacto_critic_loss", net.desc, None, bb.desc, 0.0, 0, ws.data_ptr(), nbytes, npart, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    f=ws.view(torch.float32).cpu().numpy()
    def mat(name, rows, cols, start=0): o_=offs[name]//4; return f[o_+start*cols:o_+(start+rows)*cols].reshape(rows,cols)
    x0=mat('UA0',R,16,R)[:, :2]; a1=mat('UA1',R,64,R); a2=mat('UA2',R,64,R); a3=mat('A3',R,64)
    xn=(b.xa-critic.in_center)/critic.in_half
    err=lambda g,r: np.abs(g-r).max()/max(1e-9,np.abs(r).max())
    # oracle activations: acts[0]=input(normalised), acts[1..3]
    print(trial, "x0 %.1e a1 %.1e a2 %.1e a3 %.1e"%(err(x0,xn),err(a1,acts[1]),err(a2,acts[2]),err(a3,acts[3])),
          "DEL", np.abs(mat('DEL',R,1)[:,0] - (-2*(b.v_bar - o[:,0]))).max())

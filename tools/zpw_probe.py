import sys; sys.path.insert(0,'.')
import torch
from paper_2006_10226_b200 import PackedConv2d
from workloads import gen
from workloads.shapes import resnet50_unique
c=[c for c in resnet50_unique() if c.name=="layer2.0.conv1"][0]
g=gen.rng(11); B=256
A=torch.from_numpy(gen.rand_q(g,(B,c.H,c.W,c.C),"u8")).cuda()
for zpw, wd in ((121,"u8"),(0,"s8")):
    W=torch.from_numpy(gen.rand_q(g,(c.K,c.R,c.S,c.C),wd, -127 if wd=="s8" else None, 127 if wd=="s8" else None)).cuda()
    op=PackedConv2d(B,c.H,c.W,c.C,W,None,128,zpw,0.02,[0.004],dict(scale=2.0,zero_point=0,dtype="u8",rounding="upward",relu=True),c.stride,c.pad)
    y=op(A)
    for _ in range(3): op(A,out=y)
torch.cuda.synchronize()

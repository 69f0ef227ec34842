import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
from synth import gen
cfg = gen.config("C2")
X = torch.from_numpy(cfg["X"]).cuda()
G.ggm_gram_eig(X, 0, 50); torch.cuda.synchronize()
G.ggm_gram_eig(X, 0, 50); torch.cuda.synchronize()

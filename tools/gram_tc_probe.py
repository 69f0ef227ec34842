"""Eigenvalue error of the tensor-core chunk Gram vs the oracle by fp32 slice length (GGM_GRAM_TC_SLICE)."""
import os, sys
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
import oracle as O
import paper_2407_19892_b200 as G
from test_gpu_sparse_input import _sparse_counts, _csr
for shape in [(20000,300),(300,9000)]:
    X=_sparse_counts(11+shape[0],*shape,keep=0.2); rp,c,v=_csr(X)
    Eo=O.gram_eig(X,0,12)[1]
    print(shape, 'slice', os.environ.get('GGM_GRAM_TC_SLICE'), 'max rel', np.max(np.abs(G.ggm_gram_eig_csr(rp,c,v,shape[1],12)[1].cpu().numpy()-Eo)/Eo))

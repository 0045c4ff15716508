import sys
sys.path.insert(0, '.')
import torch
from paper_1912_02767_b200.admm import MaxCutADMM
from workloads.generators import maxcut_graph
L = maxcut_graph(n=2000, p_edge=0.01, seed=501)
s = MaxCutADMM(L)
print(s.step(), flush=True)

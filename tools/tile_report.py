import sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ctypes as C
import bench
from paper_2006_04984_b200 import abi, api
for (name, c, h, w, k, st) in bench.RESNET50_3X3:
    ls = api.layer_shape(32, c, h, w, k, 3, 3, st, st, 1, 1)
    f = torch.zeros(ls.filter_dims(), dtype=torch.int8, device='cuda')
    pl = api.ConvPlan(ls, f, abi.CHECK_FIC)
    i = pl.info
    units = i.m_tiles * i.n_tiles
    print(name, 'block_n', i.block_n, 'n_tiles', i.n_tiles, 'm_tiles', i.m_tiles, 'units', units, 'b_res', i.b_resident, 'smem', i.smem_bytes)

import sys; sys.path.insert(0,'.')
import numpy as np, bench, paper_0805_1827_b200 as E
from paper_0805_1827_b200 import backend as G
from paper_0805_1827_b200.packs import pack_market, RulePack
cfg = bench.CONFIGS['c4']
p, s = bench.build_objects(cfg, E)
mp = pack_market(p, s)
rp = RulePack.european(False)
for mode in ('fast', 'parity'):
    st = G.price_blocks(mp, rp, 1 << 18, 1827, mode=mode)
    print(mode, E.pool_moments(st[:,0], st[:,1], st[:,2]))

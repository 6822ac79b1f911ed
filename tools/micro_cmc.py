import sys
sys.path.insert(0, '.')
from tests import _cases as CS
from paper_0805_1827_b200 import backend as G
d = int(sys.argv[1]) if len(sys.argv) > 1 else 10
mode = sys.argv[2] if len(sys.argv) > 2 else "parity"
p, sp = CS.maxcall(d)
mp = CS.packs(p, sp)
rp = CS.random_stumps(d, 9, 100, seed=3, lo=100, hi=200)
for _ in range(2):
    G.price_blocks(mp, rp, 1 << 22, 7, mode=mode)

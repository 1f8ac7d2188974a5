import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import gen
from oracle import memdet_oracle as O
for m, nb in [(256, 1), (512, 2), (768, 3), (700, 1), (700, 2), (700, 3), (1024, 4), (1000, 4)]:
    a = gen.spd_wishart(m, m, seed=100 + m, shift=1e-2)
    ref, info = O.memdet_cholesky(a, nb)
    try:
        res = eng.memdet_cholesky(a, num_blocks=nb, out_of_core=True)
    except Exception as e:
        print(m, nb, "ERR", e); continue
    err = np.abs(res.prefix - ref) / np.maximum(1, np.abs(ref))
    bad = np.nonzero(err > 1e-10)[0]
    print(m, nb, "maxerr %.2e" % err.max(), "first bad", bad[:1], "info", res.info.ooc_blocks, res.info.ooc_block,
          res.info.ooc_reads, res.info.ooc_writes, (info.blocks_read, info.blocks_written))

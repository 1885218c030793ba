import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests")); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np
import paper_2602_10378_b200 as fk
from paper_2602_10378_b200 import _native as N
import oracle as O
port = O.get("port")
from test_gpu_parity import _mixture_inputs
tr = _mixture_inputs(port, 4096, 16)[0]
splits, flush = int(sys.argv[1]), int(sys.argv[2])
c = fk.Context([0]); c.set_option(N.OPT_SPLITS, splits); c.set_option(N.OPT_FLUSH_TILES, flush)
s = fk.score_flash(tr, 1.5, ctx=c).values
print("OK", splits, flush, flush=True)

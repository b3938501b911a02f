"""Write instance-file fixtures with the REAL reference (cqksolve/io.py) so
tests/test_io.py can check byte-identical writes and identical reads.

Run in the builder container (the reference is not on the GPU box):
  PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py
"""
import os

import numpy as np
from cqksolve import CqkInstance, SimplexInstance, gen_cqk, gen_simplex_y, write_instance

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
os.makedirs(OUT, exist_ok=True)
inst = gen_cqk("cqk-weakly-correlated", 37, 5)
write_instance(os.path.join(OUT, "weak37.cqk"), inst)
write_instance(os.path.join(OUT, "weak37.cqkb"), inst, binary=True)
box = CqkInstance(d=np.array([1.0, 2.0]), a=np.array([0.0, -1.5]), b=np.array([1.0, 0.5]),
                  l=np.array([-np.inf, 0.0]), u=np.array([np.inf, 1.0]), r=0.75)
write_instance(os.path.join(OUT, "inf2.cqk"), box)
write_instance(os.path.join(OUT, "inf2.cqkb"), box, binary=True)
y = gen_simplex_y("simplex-n01", 23, 3)
write_instance(os.path.join(OUT, "n01_23.spx"), SimplexInstance(y=y, r=1.5))
write_instance(os.path.join(OUT, "n01_23.spxb"), SimplexInstance(y=y, r=1.5), binary=True)
print(sorted(os.listdir(OUT)))

"""Development aid: run one (l, f, n) case on the GPU and compare with the reference."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1111_3297_b200 as E
from oracle.oracle import Reference
l, f, n = (int(x) for x in sys.argv[1:4])
tm = len(sys.argv) > 4 and sys.argv[4] == "test"
p = E.validate_params(l, f, n, test_mode=tm)
g, st = E.context(0).table(p)
r, rc, _ = Reference().run_sieve(l, f, n, test_mode=tm)
print("count", st.prime_count, rc, "eq", np.array_equal(g, r), "tiles", st.tiles, "logS", st.log_tile, "waves", st.waves)

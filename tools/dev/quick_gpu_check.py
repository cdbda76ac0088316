"""Ad-hoc GPU parity probe (development aid): GPU vs reference on small cases + cfg3."""
import hashlib, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1111_3297_b200 as E
from oracle.oracle import Reference, Restated

R = Reference(); O = Restated()
ctx = E.context(0)
cases = [(10, 2048, 4, False), (12, 4096, 8, False), (4, 2048, 4, True), (10, 6, 1, False), (16, 3, 5, True),
         (13, 100, 300, True), (17, 9000, 64, False), (20, 523776, 16, False), (18, 2**30, 40, False),
         (12, 2**40, 1000, False), (16, 2**45, 200, False), (13, 2**46 + 12345, 3001, False), (20, 2**41, 600, False)]
ok = True
for l, f, n, tm in cases:
    p = E.validate_params(l, f, n, test_mode=tm)
    t0 = time.time(); g, st = ctx.table(p); t1 = time.time()
    r, rc, _ = R.run_sieve(l, f, n, test_mode=tm)
    same = np.array_equal(g, r)
    ok &= same and st.prime_count == rc
    print(f"({l},{f},{n}) gpu={st.prime_count} ref={rc} table_eq={same} tiles={st.tiles} logS={st.log_tile} {t1-t0:.3f}s", flush=True)
for l, n in [(17, 64), (12, 50), (20, 64)]:
    p = E.validate_params(l, 0, n, allow_overlap=True)
    g, st = ctx.table(p)
    r, rc = R.f0_table(l, n)
    same = np.array_equal(g, r); ok &= same and st.prime_count == rc
    print(f"f0 ({l},0,{n}) gpu={st.prime_count} ref={rc} eq={same}", flush=True)
for (l, f, n, pin) in [(20, 523776, 1024, 77449842), (21, 67106816, 4096, 516358044), (22, 137438949376, 8192, 1652382527)]:
    p = E.validate_params(l, f, n)
    for k in range(2):
        st = ctx.count(p)
        print(f"cfg l={l} count={st.prime_count} pin={pin} ok={st.prime_count==pin} total={st.total_s*1e3:.2f}ms init={st.init_s*1e3:.2f}ms tiles={st.tiles} waves={st.waves} retries={st.retries}", flush=True)
    ok &= st.prime_count == pin
print("ALL_OK" if ok else "MISMATCH")

export PYTHONUNBUFFERED=1
cat > /tmp/r.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import paper_1111_3297_b200 as E
ctx = E.Context(0)
for (l,f,n) in [(20,0,4096)]:
    p = E.validate_params(l, f, n, allow_overlap=True)
    try:
        st = ctx.count(p)
        print(l,f,n,"count", st.prime_count, flush=True)
    except Exception as e:
        print(l,f,n,"ERR", e, flush=True); break
PY
ERATO_GPU_SO=paper_1111_3297_b200/liberato_gpu_debug.so CUDA_LAUNCH_BLOCKING=1 timeout 120 python /tmp/r.py > gpurun_out/dbg.txt 2>&1; head -c 3000 gpurun_out/dbg.txt

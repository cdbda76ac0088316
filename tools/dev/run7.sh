export PYTHONUNBUFFERED=1
CFGS="5" bash tools/dev/run_var.sh 2>&1

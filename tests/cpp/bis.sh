gcc -shared -fPIC -o /tmp/segv.so tests/cpp/segv_trace.c
run() { echo "== $1 | $2"; env $2 timeout 100 python -c "
import sys; sys.path.insert(0,'.')
$1
r = sk.run_bench(workers=[1, 2], steps=2, batch=8, width=8, layers=2, in_dim=4, out_dim=2, seed=3)
print('ok')
" 2>&1 | c++filt | tail -22; }
run "import numpy; import paper_1710_04162_b200 as sk" "LD_PRELOAD=/tmp/segv.so"
run "import numpy; import paper_1710_04162_b200 as sk" "OPENBLAS_NUM_THREADS=1"
run "import numpy; import paper_1710_04162_b200 as sk" "MALLOC_CHECK_=3"

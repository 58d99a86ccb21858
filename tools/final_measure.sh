#!/usr/bin/env bash
# End-of-round measurement on one B200 (run from the repo root under gpurun):
# GPU test suite, the bench line and the reference arm, the ncu launch list of
# the bench, full ncu captures of the headline gather and the C5 pair GEMM.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1
tail -2 gpurun_out/final_gpu_tests.log
python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 200 gpurun_out/final_bench.json
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; tail -c 200 gpurun_out/final_bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-c3 --no-c4 --no-cpu-baseline > gpurun_out/final_bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_rows_kernel -s 4 -c 1 \
    -o gpurun_out/final_gather python bench.py --steps 3 --warmup 3 --no-c3 --no-c4 --no-cpu-baseline --no-sgd > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:persistent -s 7 -c 1 \
    -o gpurun_out/final_gemm_pair python tools/diag/diag_c5.py 4 > /dev/null 2>&1
ls gpurun_out/

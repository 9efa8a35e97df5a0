#!/bin/bash
# tests of the Newton path, the bench line, then the ncu evidence
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inversion.py -q -m gpu -p no:cacheprovider -k "newton or cfg0 or ldlt or cfg1_full or cached" > gpurun_out/t_newton.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_cfg1.log 2>&1; echo "bench rc=$?"
bash tools/prof_round2.sh > gpurun_out/prof2.log 2>&1; echo "prof rc=$?"

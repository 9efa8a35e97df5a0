#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "rank_trunc" > gpurun_out/t_rrqr2.log 2>&1; echo "rrqr tests rc=$?"
timeout 300 python tools/rrqr_time.py 16384 6000 3000 > gpurun_out/rrqr_big2.log 2>&1; echo "rrqr time rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_ref.log 2>&1; echo "ref rc=$?"
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 > gpurun_out/r02_bench_cfg4.log 2>&1; echo "cfg4 rc=$?"

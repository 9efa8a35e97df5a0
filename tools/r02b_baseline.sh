#!/bin/bash
# round-2 (second session) baseline: GPU tests + default bench line
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r02b_gputests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b_bench.log 2>&1; echo "bench rc=$?"

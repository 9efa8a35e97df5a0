#!/bin/bash
# instrumented build (per-phase cycle counters in the Gauss-Jordan cluster panel), one
# inversion at n = 16384 and 4096; restores the normal build afterwards
LYAP_NVCC_EXTRA=-DLYAP_PANEL_PROF python -c "import paper_2510_02126_b200.build as b; b.build(force=True)" > gpurun_out/pp_build.log 2>&1
timeout 300 python tools/inv_once.py 16384 2 > gpurun_out/pp_16k.log 2>&1
timeout 300 python tools/inv_once.py 4096 2 > gpurun_out/pp_4k.log 2>&1

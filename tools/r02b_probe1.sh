#!/bin/bash
# new Newton update kernel: A-sequence tests + breakdown at 16384/4096; instrumented GJE panel
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inversion.py -q -m gpu -p no:cacheprovider -k "newton or cached or cfg0" > gpurun_out/p1_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python tools/aseq_breakdown.py 16384,4096 > gpurun_out/p1_aseq.log 2>&1; echo "aseq rc=$?"
LYAP_LIB=$PWD/paper_2510_02126_b200/prof/liblyapir_prof.so timeout 300 python tools/inv_once.py 16384 2 > gpurun_out/p1_pp16k.log 2>&1; echo "pp rc=$?"
LYAP_LIB=$PWD/paper_2510_02126_b200/prof/liblyapir_prof.so timeout 300 python tools/inv_once.py 4096 2 > gpurun_out/p1_pp4k.log 2>&1
LYAP_LIB=$PWD/paper_2510_02126_b200/prof/liblyapir_prof.so timeout 300 python tools/eig_sizes.py 900,400 > gpurun_out/p1_eig.log 2>&1

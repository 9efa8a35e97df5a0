#!/bin/bash
# panel phase cycles (instrumented library), then correctness + timings of the implicit-pivoting sweep
P=$PWD/paper_2510_02126_b200/prof/liblyapir_prof.so
LYAP_LIB=$P timeout 120 python tools/gje_ip_check.py 1024,4096 fp16 2>&1 | tail -8
LYAP_GJE_IP_NT=1024 LYAP_LIB=$P timeout 120 python tools/gje_ip_check.py 16384 fp16 2>&1 | tail -4
LYAP_GJE_IP_NT=512 LYAP_GJE_IP_RPT=2 LYAP_LIB=$P timeout 120 python tools/gje_ip_check.py 16384 fp16 2>&1 | tail -4
timeout 300 python tools/gje_ip_check.py 1024,2048,4096,8192 fp16,bf16,fp32 2>&1 | tail -14
timeout 200 python tools/aseq_time.py 1024,2048,4096,16384
LYAP_GJE_IP_NT=512 LYAP_GJE_IP_RPT=2 timeout 200 python tools/aseq_time.py 16384

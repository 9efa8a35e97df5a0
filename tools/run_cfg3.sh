export LYAP_VERBOSE=1 CHECK=1
NEWTON_COLS=8192 WORK_COLS=10240 timeout 900 python tools/explore_cfg.py cfg3 fp16 4096 > gpurun_out/e3_fp16.log 2>&1; echo "fp16 rc=$?"
NEWTON_COLS=14336 WORK_COLS=16384 timeout 1500 python tools/explore_cfg.py cfg3 fp32 6144 > gpurun_out/e3_fp32.log 2>&1; echo "fp32 rc=$?"

export LYAP_RRQR_BLOCKED=1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/rrqr_time.py 3000 700 120 > gpurun_out/san_rrqr.log 2>&1; echo "rrqr rc=$?"
unset LYAP_RRQR_BLOCKED
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/qr_once.py 9000 300 > gpurun_out/san_qr.log 2>&1; echo "qr rc=$?"
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_families.py -q -m gpu -p no:cacheprovider -k "cfg2_family_parity and 10-fp16 or stagnation_path_parity and chol" > gpurun_out/san_fam.log 2>&1; echo "fam rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/t_all3.log 2>&1; echo "all rc=$?"

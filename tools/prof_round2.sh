#!/bin/bash
# Round-2 ncu evidence (run under gpurun, one GPU): the launch list of the benched configs[1]
# solve (duration only) and full captures of the kernels the bench line names.
# Each command first runs plainly (it must exit 0), then once under ncu.
set -u
O=gpurun_out
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_cfg1.csv \
    python tools/profile_solve.py cfg1 > $O/ncu_launches.log 2>&1 || echo "launch list failed"
run() {   # name, kernel regex, skip, count, command...
    local name=$1 pat=$2 skip=$3 cnt=$4; shift 4
    "$@" > $O/plain_$name.log 2>&1 || { echo "$name: plain run failed"; return; }
    ncu --set full --clock-control none --import-source on -k regex:"$pat" -s "$skip" -c "$cnt" \
        -o $O/r02_$name -f "$@" > $O/ncu_$name.log 2>&1 || echo "$name: ncu failed"
}
run tridiag_cfg1 'tridiag_w_kernel' 20 1 python tools/profile_solve.py cfg1
run update16k 'newton_update_row' 2 1 python tools/aseq_time.py 16384
run tcgemm16k 'tc_gemm_persistent' 40 1 python tools/inv_once.py 16384 2
run qrgrid 'qr_panel_reg_kernel<true>|qr_panel_reg_kernelILb1' 10 1 python tools/qr_once.py 16384 1100
run rrqr3 'rrqr3_kernel' 3 1 python tools/rrqr_time.py 16384 3000 700
ls -la $O/*.ncu-rep

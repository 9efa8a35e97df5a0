#!/bin/bash
# ncu captures behind the round-1 notes in profiles/ (run under gpurun, one GPU).
# Each command first runs plainly (it must exit 0), then once under ncu.
set -u
O=gpurun_out
mkdir -p $O
run() {   # name, kernel regex, skip, count, command...
    local name=$1 pat=$2 skip=$3 cnt=$4; shift 4
    "$@" > $O/plain_$name.log 2>&1 || { echo "$name: plain run failed"; return; }
    ncu --set full --clock-control none --import-source on -k regex:"$pat" -s "$skip" -c "$cnt" \
        -o $O/prof_$name -f "$@" > $O/ncu_$name.log 2>&1 || echo "$name: ncu failed"
}
run gje16k 'gje_panel_cluster' 512 2 python tools/inv_once.py 16384 2
run xabove16k 'gje_xabove' 512 2 python tools/inv_once.py 16384 2
run rrqr 'rrqr2_kernel' 2 1 python tools/rrqr_time.py 4096 1400 400
run trid2400 'tridiag_kernel' 2 1 python tools/eig_sizes.py 2400
ls -la $O/*.ncu-rep

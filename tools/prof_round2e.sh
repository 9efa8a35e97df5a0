#!/bin/bash
# Round-2 (third session, final state) ncu evidence, run under gpurun on one GPU: the default bench line,
# the launch list of the benched configs[1] solve and of one n = 16384 inversion (duration
# only), and full captures of the implicit-pivoting inversion's kernels.  Every command runs
# plainly first (it must exit 0), then once under ncu.
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/r02e_bench_cfg1.json 2> $O/r02e_bench_cfg1.err || echo "bench failed"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02e_launches_cfg1.csv \
    python tools/profile_solve.py cfg1 > $O/ncu_launches_c.log 2>&1 || echo "launch list failed"
ncu --metrics gpu__time_duration.sum --clock-control none -s 1600 -c 1800 --csv --log-file $O/r02e_launches_inv16k.csv \
    python tools/inv_once.py 16384 2 > $O/ncu_launches_inv.log 2>&1 || echo "inversion launch list failed"
run() {   # name, kernel regex, skip, count, command...
    local name=$1 pat=$2 skip=$3 cnt=$4; shift 4
    "$@" > $O/plain_$name.log 2>&1 || { echo "$name: plain run failed"; return; }
    ncu --set full --clock-control none --import-source on -k regex:"$pat" -s "$skip" -c "$cnt" \
        -o $O/r02e_$name -f "$@" > $O/ncu_$name.log 2>&1 || echo "$name: ncu failed"
}
run ip_panel16k 'gje_ip_panel_kernel' 100 1 python tools/inv_once.py 16384 1
run ip_panel1k 'gje_ip_panel_kernel' 20 1 python tools/inv_once.py 1024 1
run ip_fused16k 'rank32_fused_kernel' 100 1 python tools/inv_once.py 16384 1
run ip_fused1k 'rank32_fused_kernel' 20 1 python tools/inv_once.py 1024 1
run ip_prep16k 'gje_ip_outer_prep' 4 1 python tools/inv_once.py 16384 1
run tcgemm16k 'tc_gemm_persistent' 20 1 python tools/inv_once.py 16384 1
run tcgemm_rest16k 'tc_gemm_kernel' 10 1 python tools/inv_once.py 16384 1
run update16k 'newton_update' 2 1 python tools/aseq_time.py 16384
run tridiag_cfg1 'tridiag_w_kernel' 20 1 python tools/profile_solve.py cfg1
ls -la $O/r02e_*.ncu-rep

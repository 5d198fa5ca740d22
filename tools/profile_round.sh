set -x
# One GPU call: the profile set of a round (ncu captures only after the plain runs pass).
D=gpurun_out/${ROUNDTAG:-r02}; mkdir -p $D
python tools/apply_once.py C2 - 1 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cutp|k_tile2|k_uncw" -c 3 -o $D/ncu_full_c2 python tools/apply_once.py C2 - 1 > $D/ncu_full_c2.log 2>&1
python tools/ncu_traffic.py $D/ncu_full_c2.ncu-rep C2 "k_cutp<4>=k_cutp" "k_tile2<4,0> + k_uncw<4,8>=k_tile2|k_uncw" >> $D/ncu_full_c2.log 2>&1
python tools/apply_once.py C5 - 1 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cut|k_uncw" -c 2 -o $D/ncu_full_c5 python tools/apply_once.py C5 - 1 > $D/ncu_full_c5.log 2>&1
python tools/ncu_traffic.py $D/ncu_full_c5.ncu-rep C5 "k_cut<6>=k_cut" "k_uncw<6>=k_uncw" >> $D/ncu_full_c5.log 2>&1
cp profiles/ncu_traffic.json $D/
timeout 900 python bench.py --steps 40 > $D/bench_c2.json 2> $D/bench_c2.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-csr --no-cpu-baseline > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-csr --no-cpu-baseline > $D/ncu_launch.log 2>&1
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-csr --no-cpu-baseline --cg 50 > $D/bench_c5_cg.json 2> $D/bench_c5_cg.err
timeout 900 python bench.py --config C4 --steps 10 --warmup 3 --no-csr --no-cpu-baseline --cg 50 > $D/bench_c4_cg.json 2> $D/bench_c4_cg.err
timeout 900 python tools/sweep.py > $D/sweep.jsonl 2> $D/sweep.err
timeout 900 python tools/h1_bench.py C2 C5 > $D/h1.jsonl 2> $D/h1.err
timeout 900 python tools/plane_sweep.py > $D/plane_sweep.jsonl 2> $D/plane_sweep.err
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
for c in 'C2 -' 'C3 1' 'C3 2' 'C5 -' 'C3 8'; do python tools/apply_once.py $c 1 > /dev/null 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv python tools/apply_once.py $c 1 2>/dev/null | grep -v '^==' ; done > $D/flops.csv

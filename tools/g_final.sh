#!/bin/bash
# round-2 final evidence: full GPU suite (+ threshold sweep log, smoke), sanitizers, bench, sweep, ncu
T=${1:-r2f}
D=gpurun_out/prof_$T; mkdir -p $D
export PYTHONUNBUFFERED=1 FTGEMM_FP_SWEEP_OUT=$D
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > $D/pytest.txt; tail -3 $D/pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
mkdir -p gpurun_out/sanitize; bash tools/g_sanitize.sh > /dev/null 2>&1; cp gpurun_out/sanitize/*.txt $D/ 2>/dev/null; cat $D/summary.txt
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 200 $D/bench.json
timeout 300 python bench.py --steps 20 --warmup 5 > $D/bench20.json 2> $D/bench20.err; tail -c 200 $D/bench20.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --backend gloo --steps 6 --warmup 3 --no-sweep > $D/multi_gloo.json 2> $D/multi_gloo.err; tail -c 200 $D/multi_gloo.json
timeout 1500 python tools/sweep.py --out $D/sweep.json > $D/sweep.log 2>&1; tail -1 $D/sweep.log | cut -c1-100
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 20 --warmup 3 --no-sweep --cpu-seconds 1 > $D/ncu_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_ft python tools/prof_run.py bf16 8192 2 > $D/p1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_off python tools/prof_run.py bf16 8192 0 > $D/p2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:encode_ab -s 1 -c 1 -o $D/encode_ab python tools/prof_run.py bf16 8192 2 > $D/p3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_k128 python tools/prof_shape.py bf16 16384 16384 128 2 > $D/p4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:simt_ftgemm -s 1 -c 1 -o $D/simt_ft python tools/prof_run.py f32_simt 4096 2 > $D/p5.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_a python tools/prof_fused.py 8192 8192 8192 > $D/p6.log 2>&1
# in-kernel A encode timeline (needs the -DFTGEMM_EXP_FA_TRACE build: libftgemm_fa_trace.so)
for f in 0 1; do FUSE=$f FTGEMM_LIB=paper_2305_01024_b200/libftgemm_fa_trace.so timeout 200 python tools/fa_trace.py bf16 8192 8192 8192 >> $D/fa_trace.txt 2>&1; done
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back limit)
python tools/profile_summary.py $T $D/launches.csv $D/fused_ft.ncu-rep $D/fused_off.ncu-rep $D/encode_ab.ncu-rep $D/fused_k128.ncu-rep $D/simt_ft.ncu-rep $D/fused_a.ncu-rep > $D/summary_profiles.log 2>&1
python tools/sweep_md.py $D/sweep.json profiles/${T}_sweep.md >> $D/summary_profiles.log 2>&1
mkdir -p $D/profiles; cp profiles/${T}_* profiles/ncu_traffic.json $D/profiles/ 2>/dev/null
rm -f $D/*.ncu-rep
echo done

#!/bin/bash
# Round-2 closing GPU pass (r02k): full GPU suite, bench (with cpu_baseline), reference arm,
# launch list of one op-sweep step, ncu --set full of the attention kernels, of the index /
# merge kernels and of the GEMM (pair and single-CTA), pretrain launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph --interp-images 0 --pretrain-batch 0 --tiny-batch 0 --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'attn_(fwd|bwd_q|bwd_kv)_kernel' -s 5 -c 5 \
  -o gpurun_out/prof_attn -f $B > gpurun_out/ncu_full.log 2>&1; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'pool_fwd_v3|pool_bwd_v3|select_topk|assign_kernel|pool_topk|seg_sort|nbr_v2_kernel|attn_qrec|attn_krec' -s 9 -c 9 \
  -o gpurun_out/prof_merge -f $B > gpurun_out/ncu_full2.log 2>&1; echo "ncu index/merge rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_pair -f python tools/gemm_one.py 16768 4096 1024 fwd > gpurun_out/ncu_g1.log 2>&1; echo "ncu gemm pair rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_gelu -f python tools/gemm_one.py 41920 2048 512 gelu > gpurun_out/ncu_g2.log 2>&1; echo "ncu gemm gelu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pretrain_launches.csv \
  python tools/pretrain_probe.py --batch 16 --steps 1 --no-graph > gpurun_out/ncu_pretrain.log 2>&1; echo "ncu pretrain rc=$?"
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB return limit)
for r in prof_attn prof_merge prof_gemm_pair prof_gemm_gelu; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
[ -x tools/micro/pdl_gap ] && timeout 60 tools/micro/pdl_gap > gpurun_out/pdl_gap.txt 2>&1

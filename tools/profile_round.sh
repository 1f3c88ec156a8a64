#!/bin/bash
# Round profile capture on the GPU box (one GPU).  usage: bash tools/profile_round.sh <tag>
# Every ncu pass runs only after the same command exited 0 without ncu.
set -u
tag=${1:-r1}
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build_$tag.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --pairs 1 --no-cpu --no-stack > $o/plain_bench_$tag.log 2>&1 || exit 2
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --pairs 1 --no-cpu --no-stack > $o/ncu_launch_$tag.log 2>&1
for s in 0 1 2 3; do
  python tools/prof_layer.py $s 2 > $o/plain_${tag}_$s.log 2>&1 || continue
  # stages 0/1 run the one-kernel plan (1 launch per run), stages 2/3 two kernels
  if [ $s -lt 2 ]; then skip=1; cnt=1; else skip=2; cnt=2; fi
  ncu --set full --clock-control none --import-source on -k regex:"mlp_gemm_kernel|fused_mlp_kernel" \
      -s $skip -c $cnt -o $o/full_stage$s -f python tools/prof_layer.py $s 2 > $o/ncu_full_${tag}_$s.log 2>&1
done
for s in 2 3; do python tools/trace_layer.py $s > $o/trace_${tag}_$s.log 2>&1; done
python tools/trace_fused.py 96 200704 > $o/trace_${tag}_0.log 2>&1
python tools/trace_fused.py 192 50176 > $o/trace_${tag}_1.log 2>&1

# north-star stage: Swin-B b128 stage 3 layer (C = 512, T = 25088), both kernels
python tools/layer_sweep.py 512 25088 3 > $o/plain_swinb3_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mlp_gemm_kernel -s 6 -c 2 -o $o/full_swinb3 -f \
    python tools/layer_sweep.py 512 25088 3 > $o/ncu_full_swinb3_$tag.log 2>&1
python tools/stack_bench.py 4 3 --steps 10 > $o/stack_$tag.log 2>&1

# FasterTransformer-layout arm (NEXT-1): launch list with DRAM bytes
python tools/prof_ft.py gelu 1 > $o/plain_ft_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $o/ft_launches_$tag.csv python tools/prof_ft.py gelu 1 > $o/ncu_ft_$tag.log 2>&1
# attention half (NEXT-3 / NEXT-4), Swin-T b64 stage 0: op #1, QKV GEMM + op #2, attention core
python tools/attn_one.py 0 2 > $o/plain_attn_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"attn_core|op1_kernel|mlp_gemm_kernel" -s 3 -c 3 \
    -o $o/full_attn0 -f python tools/attn_one.py 0 2 > $o/ncu_full_attn_$tag.log 2>&1
# configs[0]: one 7x7 window, the one-launch plan (small_mlp.cuh)
python tools/prof_layer.py 768x49 3 > $o/plain_config0_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:small_mlp -s 2 -c 1 -o $o/full_config0 -f \
    python tools/prof_layer.py 768x49 3 > $o/ncu_full_config0_$tag.log 2>&1
python tools/trace_small.py 768 49 > $o/trace_${tag}_config0.log 2>&1
# bring-back budget (gpurun merges <= 64 MiB): raw + source CSV exports of every capture,
# the .ncu-rep only for the dominant stage-0 kernel
for s in 0 1 2 3 swinb3 attn0 config0; do
  [ -f $o/full_stage$s.ncu-rep ] || [ -f $o/full_$s.ncu-rep ] || continue
  [ -f $o/full_$s.ncu-rep ] && mv $o/full_$s.ncu-rep $o/full_stage$s.ncu-rep
  ncu -i $o/full_stage$s.ncu-rep --page raw --csv > $o/full_stage${s}_raw.csv 2>/dev/null
  ncu -i $o/full_stage$s.ncu-rep --page details --csv > $o/full_stage${s}_details.csv 2>/dev/null
  [ "$s" != 0 ] && rm -f $o/full_stage$s.ncu-rep
done
du -sh $o
echo done

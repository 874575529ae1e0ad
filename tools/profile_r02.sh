# Round-2 profiles (run on the GPU box from the repo root; each ncu pass only after its plain run exits 0).
#  1. the launch list of the bench command itself over its timed steps (MPS_BENCH_PROFILE_RANGE=1
#     brackets them with cudaProfilerStart/Stop; per-launch times are cold-cache and serialised);
#  2. ncu --set full of the default K1 (site_gemm3m_kernel, 3M + sum planes) at C3 mode 30, one lane;
#  3. the same for the K2+K3 draw kernel at mode 30;
#  4. ncu --set full of the small-chain kernel (v2) at C2, n = 100 (the whole chain in one launch).
set -x
P="ncu --clock-control none"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_plain.jsonl 2> gpurun_out/r02_bench_plain.err && \
MPS_BENCH_PROFILE_RANGE=1 timeout 900 $P --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02_launches_bench_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 python tools/profile_step.py --lanes 1 > gpurun_out/r02_ps_plain.log 2>&1 && \
timeout 600 $P --profile-from-start off --set full --import-source on -k regex:site_gemm3m -s 30 -c 1 \
  -o gpurun_out/r02_k1_c3_mode30 python tools/profile_step.py --lanes 1 > /dev/null 2>&1
timeout 600 $P --profile-from-start off --set full --import-source on -k regex:displace_draw -s 30 -c 1 \
  -o gpurun_out/r02_draw_c3_mode30 python tools/profile_step.py --lanes 1 > /dev/null 2>&1
timeout 300 python tools/profile_step.py --config c2 > gpurun_out/r02_ps_c2.log 2>&1 && \
timeout 600 $P --profile-from-start off --set full --import-source on -k regex:small_chain -c 1 \
  -o gpurun_out/r02_small_chain2_c2 python tools/profile_step.py --config c2 > /dev/null 2>&1
ls -la gpurun_out/ | grep r02

set -x
P="ncu --profile-from-start off --clock-control none"
timeout 300 python tools/profile_step.py > gpurun_out/ps_plain.log 2>&1 && \
timeout 300 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r01_launches_c3_3m_lanes2.csv python tools/profile_step.py > /dev/null 2>&1
timeout 300 python tools/profile_step.py --gemm ozaki > gpurun_out/ps_plain2.log 2>&1 && \
timeout 300 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r01_launches_c3_ozaki_lanes2.csv python tools/profile_step.py --gemm ozaki > /dev/null 2>&1
timeout 300 $P --set full --import-source on -k regex:ozaki2 -s 30 -c 1 -o gpurun_out/r01_ozaki2_c3_mode30 python tools/profile_step.py --gemm ozaki --lanes 1 > /dev/null 2>&1
timeout 300 $P --set full --import-source on -k regex:displace_draw -s 30 -c 1 -o gpurun_out/r01_draw_c3_mode30 python tools/profile_step.py --lanes 1 > /dev/null 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1.log 2>&1; tail -1 gpurun_out/torchrun1.log | cut -c1-200
ls gpurun_out/

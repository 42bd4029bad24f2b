set -x
nvidia-smi topo -m | head -8
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
tail -2 gpurun_out/bench_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
python tools/nvlink_probe.py cfg3_R4 4 > gpurun_out/nvlink_cfg3_R4.json 2> gpurun_out/nvlink.err
python tools/nvlink_probe.py cfg2_R4 4 > gpurun_out/nvlink_cfg2_R4.json 2>> gpurun_out/nvlink.err
tail -3 gpurun_out/nvlink.err
python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_rank.py -q > gpurun_out/t_multi.log 2>&1; tail -3 gpurun_out/t_multi.log
python tools/perf_probe.py cfg3_R4 2 > gpurun_out/merge_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:merge_kernel -c 6 --csv python tools/perf_probe.py cfg3_R4 2 > gpurun_out/ncu_merge.csv 2> gpurun_out/ncu_merge.err
tail -3 gpurun_out/ncu_merge.csv

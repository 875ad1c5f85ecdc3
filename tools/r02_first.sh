#!/bin/bash
# r02 first GPU pass: gpu tests, smoke, default bench, launch list of one step
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r02_gpu.txt; nproc >> gpurun_out/r02_gpu.txt; lscpu | grep "Model name" >> gpurun_out/r02_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02_ncu_launch.log 2>&1
tail -3 gpurun_out/r02_gputest.log; tail -c 1500 gpurun_out/r02_bench.json

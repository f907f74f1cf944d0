#!/bin/bash
# round-2 check: full-size parity tests, bench (N=1), host-transport N=2 self-launch, reference arm
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20) > gpurun_out/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "full_size or config3_512 or config2_256" -s > gpurun_out/t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/t1.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.log 2>&1; echo "b1 rc=$?" >> gpurun_out/b1.log
timeout 600 python bench.py --gpus 2 --transport host --n 256 --steps 5 --warmup 3 > gpurun_out/b2.log 2>&1; echo "b2 rc=$?" >> gpurun_out/b2.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r1.log 2>&1; echo "r1 rc=$?" >> gpurun_out/r1.log

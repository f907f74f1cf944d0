mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_p2.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pipe_yinv|k_pipe_xinv" -s 2 -c 2 -o gpurun_out/p2prof python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_p2.log 2>&1; echo "ncu rc=$?"

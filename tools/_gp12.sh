python -m pytest tests/test_gpu_dist.py -q -x -k "gmres" > gpurun_out/t12.log 2>&1; echo "dist rc=$?"; tail -c 1500 gpurun_out/t12.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --force-dist --steps 2 --warmup 1 --scale 0.5 > gpurun_out/b12.log 2>&1; echo "fd rc=$?"; tail -c 1200 gpurun_out/b12.log

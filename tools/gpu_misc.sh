mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "mahalanobis_sort" -p no:cacheprovider > gpurun_out/misc_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/misc_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/misc_torchrun.json 2> gpurun_out/misc_torchrun.err
echo "torchrun rc=$?" >> gpurun_out/misc_torchrun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/misc_torchrun_ref.json 2>> gpurun_out/misc_torchrun.err
echo "torchrun ref rc=$?" >> gpurun_out/misc_torchrun.err

# end-of-session check: GPU suite, default bench, 2-rank bench (ranks sharing the GPU), reference arm, smoke
set -x
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python bench.py > gpurun_out/fc_b1.json 2> gpurun_out/fc_b1.err; tail -c 600 gpurun_out/fc_b1.json; tail -3 gpurun_out/fc_b1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/fc_b2.json 2> gpurun_out/fc_b2.err; echo rc=$?; tail -c 300 gpurun_out/fc_b2.json
timeout 300 python bench.py --impl reference > gpurun_out/fc_r1.json 2>&1; tail -c 300 gpurun_out/fc_r1.json
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2

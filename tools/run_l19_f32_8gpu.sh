#!/bin/bash
# l = 19 in fp32 storage, sharded (the folded quarter table: 2 x 192 GiB, i.e. >= 4 GPUs; 8 here):
# the paper's first external-memory point, 0.791389 (183,431 s on disk).
# DESIGN.md §9c.   NPROC=4 bash tools/run_l19_f32_8gpu.sh
# Integer offsets on (R23; sharded since the end of round 2): fp32 alone gave 0.790656 at l = 18
# vs the paper's 0.790668, with offsets 0.790666.
python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NPROC:-8} --master-addr 127.0.0.1 \
    --master-port 29621 tools/converge_sharded.py --ell 19 --dtype f32 --offsets 1 --every 20 "$@"

#!/bin/bash
# l = 19 in fp32 storage on 8 B200 (sharded half table, 137 GB per GPU): the paper's first
# external-memory point, 0.791389 (183,431 s on disk).  DESIGN.md §9.
python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29621 tools/converge_sharded.py --ell 19 --dtype f32 --every 20 "$@"

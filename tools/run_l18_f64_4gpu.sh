#!/bin/bash
# l = 18 in fp64 storage on 4 B200 (sharded half table, 137 GB per GPU): Table 2's 0.790668
# to the sixth digit.  DESIGN.md §9.
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29620 tools/converge_sharded.py --ell 18 --dtype f64 --every 20 "$@"

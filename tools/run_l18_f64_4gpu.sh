#!/bin/bash
# l = 18 in fp64 storage, sharded (the folded quarter table by default: 2 x 96 GiB over the GPUs,
# so 2 GPUs suffice; 4 leave room), converged: Table 2's 0.790668.  DESIGN.md §9c.
#   NPROC=2 bash tools/run_l18_f64_4gpu.sh
python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NPROC:-4} --master-addr 127.0.0.1 \
    --master-port 29620 tools/converge_sharded.py --ell 18 --dtype f64 --every 20 "$@"

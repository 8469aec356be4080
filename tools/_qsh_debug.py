import faulthandler, os, sys
pass
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
from paper_2407_10925_b200.dist import create_sharded
print("r", rank, "create", flush=True)
h = create_sharded(10, dtype="f32", transport="host", symmetry=2, block_log4=5)
print("r", rank, "created", h.kernel_in_use, flush=True)
h.sweep(2)
print("r", rank, "swept", flush=True)
b = h.bound()
print("r", rank, "bound", b.bound, flush=True)
t = h.table(0)
print("r", rank, "table", t[:4], flush=True)
dist.barrier()
h.destroy()
print("r", rank, "destroyed", flush=True)
dist.destroy_process_group()

"""B200-native Feasible Triplet sweeps (arXiv 2407.10925): the C-ABI library liblcsb.so and its
thin Python binding.  See include/lcsb.h and DESIGN.md."""
from .lcsb import (  # noqa: F401
    BoundResult, Lcsb, LcsbError, SO_PATH, lcsb_bound, lcsb_create, lcsb_destroy,
    lcsb_required_bytes, lcsb_reset, lcsb_sweep, lcsb_table, lcsb_table_gather, load_library,
)

"""CPU oracle for the DDL all-reduce -- TEST INFRASTRUCTURE ONLY (see ddl_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It shares no code with paper_1811_12174_b200/.
"""
from .ddl_oracle import *  # noqa: F401,F403
from .ddl_oracle import (allreduce, reduce_scatter, allgather, allreduce_sampled, local_reduce,  # noqa: F401
                         naive_sum, exact_sum_f64, bf16_round, bf16_to_f32, parse_dims, validate_dims,
                         coord, group, active_blocks, schedule, block_elems, block_range, Traffic,
                         avg_scale, fold_error_bound, BadDims, LengthMismatch, EmptyBuffers, Unsupported)

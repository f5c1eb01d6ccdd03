"""wheelsieve-b200: the B200-native (sm_100a) segmented mod-6 wheel sieve.

Importing loads libwheelsieve_cuda.so (the C ABI of include/wheelsieve/gpu.h);
there is no CPU fallback."""
from .wheelsieve import (  # noqa: F401
    CountSink, Checks, Errc, Error, MemorySink, PrimeSink, Sieve, SieveConfig, SieveReport,
    SinkFailure, isqrt, partition, prime_count_bound, round_segment_span, run, run_unbounded,
    start_offsets, ceil_sqrt, value_of, coord_of, R1, R5, read_back, verify_store, PrimeStream,
    combine_checks, nccl_unique_id, plan_iteration, WorkerAssignment,
)

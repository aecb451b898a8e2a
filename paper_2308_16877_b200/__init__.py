"""B200-native approximate-region engine (HPAC-Offload hot path, arXiv 2308.16877).

The product is libhpac_b200.so (CUDA sm_100a kernels behind the C-ABI in
include/hpac_offload.h); this package is its Python host mirror.
"""
from . import abi  # noqa: F401
from .engine import (  # noqa: F401
    ArenaOverflowError, BarrierDivergenceError, ConfigError, CudaError, DirectiveError,
    GridConfig, KmeansResult, LaunchResult, Region, SimtError, UnsupportedError, WorkMapping, arena_required,
    binomial_region, blackscholes_region, iact, kmeans_region, kmeans_run, lavamd_region, make_lavamd, make_binomial_portfolio,
    make_blobs, make_bs_portfolio, mape, mcr, parse_directive, perfo, resolve_grid, run_region,
    run_region_host, synthetic_region, table_region, taf, unparse)

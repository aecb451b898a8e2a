"""Helpers to run cases through the CUDA engine (torch device buffers)."""
from __future__ import annotations

import numpy as np
import torch

from paper_2308_16877_b200 import engine as E


def dev(x):
    if x is None:
        return None
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run_case_gpu(case):
    """Returns (status, stats dict, outputs ndarray, paths ndarray, message)."""
    out = dev(case.init.copy())
    paths = torch.zeros(max(case.n, 1), dtype=torch.uint8, device="cuda")
    region = E.table_region(dev(case.inputs), dev(case.table), out, input_dims=case.in_dims,
                            output_dims=case.out_dims, encounters=dev(case.encounters),
                            accumulate=case.accumulate, barrier=case.barrier)
    try:
        lr = E.run_region(case.grid, case.n, case.mapping, region, case.spec, paths=paths)
        status, stats, msg = 0, lr.stats, ""
    except E.ArenaOverflowError as e:
        status, stats, msg = 2, {"arena_required": e.required_bytes, "arena_available": e.available_bytes}, str(e)
    except E.BarrierDivergenceError as e:
        status, stats, msg = 3, {"fail_team": e.team_id, "fail_step": e.step, "fail_missing": e.missing}, str(e)
    except E.ConfigError as e:
        status, stats, msg = 1, {}, str(e)
    torch.cuda.synchronize()
    return status, stats, out.cpu().numpy(), paths.cpu().numpy()[: case.n], msg

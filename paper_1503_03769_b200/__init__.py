"""B200-native hot path of the distributed particle PHD filter (arXiv 1503.03769).

The product is the C-ABI library ``lib/libphd.so`` (include/phd.h) built from
``csrc/`` for sm_100a; :mod:`.binding` is its thin ctypes binding.
"""
from .binding import (Filter, LocalGroup, Params, Estimate, Summary, PhdError, load, params_from, nccl_unique_id,
                      philox, philox_device, host_transport, rank_block, resample_bounds, plan_exchange, workspace_size, lib_path,
                      STAGE_PREDICTED, STAGE_RESAMPLED, EXPORTS)

__all__ = ["Filter", "LocalGroup", "Params", "Estimate", "Summary", "PhdError", "load", "params_from", "nccl_unique_id",
           "philox", "philox_device", "host_transport", "rank_block", "resample_bounds", "plan_exchange", "workspace_size", "lib_path",
           "STAGE_PREDICTED", "STAGE_RESAMPLED", "EXPORTS"]

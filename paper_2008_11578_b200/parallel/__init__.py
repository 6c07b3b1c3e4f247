"""Spatial strip decomposition across the GPUs of one node (one process per GPU,
torch.distributed / NCCL for the halo and migration traffic)."""

from .strips import DeviceStripOps, StripDriver, strip_bounds

__all__ = ["DeviceStripOps", "StripDriver", "strip_bounds"]

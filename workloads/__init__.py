"""Synthetic workloads (circuits, noise, shots) for TUSQ — inputs only, no method arithmetic."""
from .circuits import *  # noqa: F401,F403

"""Task splitting (the *hyper* ``hyper.for`` range partition), B200 engine side."""

from .partition import partition_range, round_half_up

__all__ = ["partition_range", "round_half_up"]

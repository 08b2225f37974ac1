"""Seeded synthetic message streams shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no ring layout, no pointer
formula, no checksum): it only draws message sizes, header field values and
payload bytes from a seed.  It is the one module both `oracle/` and the tests /
bench of the product path may import (task rule: "only the seeded input
generators serve both, from a module of their own").
"""
from .streams import *  # noqa: F401,F403

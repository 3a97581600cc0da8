"""CPU float64 oracle (TEST INFRASTRUCTURE ONLY -- see fbp_oracle.py header)."""
from .fbp_oracle import *  # noqa: F401,F403

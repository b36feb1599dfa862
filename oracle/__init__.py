"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY (see moe_oracle.py header)."""

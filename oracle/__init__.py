"""CPU oracle (test infrastructure only; see pnce_oracle.py header)."""

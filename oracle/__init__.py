"""CPU oracle (test infrastructure only; see gbopt_oracle.py header)."""

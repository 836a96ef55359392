"""CPU oracle package (test infrastructure only; see cpu_oracle.py)."""

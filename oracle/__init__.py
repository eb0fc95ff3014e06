"""CPU oracle for the SLIDE hot path -- test infrastructure only (see slide_oracle.py)."""

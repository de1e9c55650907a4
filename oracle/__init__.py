"""CPU oracle for parity tests -- TEST INFRASTRUCTURE ONLY (see lm_oracle.py)."""

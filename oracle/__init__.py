"""CPU oracles for parity tests -- test infrastructure only (see oracle/oracle.py)."""

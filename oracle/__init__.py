"""TEST INFRASTRUCTURE ONLY — CPU oracles (see oracle/oracle.py)."""

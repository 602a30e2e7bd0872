"""ORACLE package — test infrastructure only (see ringmix_oracle.py)."""

"""CPU oracle (test infrastructure only): see cntgw_oracle.py."""

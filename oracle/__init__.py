"""CPU oracle package -- test infrastructure only (see oracle/ssj_oracle.h)."""

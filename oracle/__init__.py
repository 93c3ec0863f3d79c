"""fp64 CPU oracle (test infrastructure only; see oracle/pdilqr_oracle.c header)."""

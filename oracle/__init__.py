"""CPU oracle of the PSSO hot path -- test infrastructure only (see psso_oracle.c)."""

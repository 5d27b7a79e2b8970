"""CPU oracle (test infrastructure only; see cpkit_oracle.cpp header)."""

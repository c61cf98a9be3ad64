"""CPU oracle of the reference AIRES hot path -- TEST INFRASTRUCTURE ONLY (see aires_oracle.h)."""

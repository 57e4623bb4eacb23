"""CPU oracle of the GLS hot path (test infrastructure only; see gls_ref.py)."""

"""TEST INFRASTRUCTURE ONLY: CPU oracle of the reference (see oracle.py)."""

"""TEST INFRASTRUCTURE ONLY: CPU oracle for the SpMV hot path (see oracle.py)."""

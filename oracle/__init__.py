"""TEST INFRASTRUCTURE ONLY: checkers for the GPU path (see ref.py)."""

"""TEST INFRASTRUCTURE ONLY: CPU checkers for the GPU sieve (see oracle.py)."""

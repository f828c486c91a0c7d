"""TEST INFRASTRUCTURE ONLY: CPU oracle of the FlashFPS hot path (see oracle.py)."""

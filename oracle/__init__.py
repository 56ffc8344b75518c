"""TEST INFRASTRUCTURE: CPU oracle for the Megopolis hot path (see oracle.py)."""

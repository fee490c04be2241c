"""TEST INFRASTRUCTURE ONLY.  See oracle/laze_port.py."""

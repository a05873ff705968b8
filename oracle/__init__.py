"""TEST INFRASTRUCTURE ONLY (the checker).  See oracle/bind.py."""

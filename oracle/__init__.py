"""TEST INFRASTRUCTURE — checkers only (see oracle/pyoracle.py); never imported by the product."""

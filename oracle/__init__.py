"""Test-only CPU oracle (see oracle/semref.py header).  Never imported by the product."""

"""Test-infrastructure oracle (see hq_oracle.py header).  Not part of the product."""

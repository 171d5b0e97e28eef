"""Test-infrastructure oracle (CPU restatement of the reference path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import
this package.  See oracle/oracle.py and oracle/gaes_oracle.c.
"""

"""Test-only CPU oracle (numpy restatement of the reference `kvrot` hot path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  The product package never does.
"""

"""Test infrastructure: CPU restatement of the reference BitSnap codec.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package, and only as the checker / CPU baseline — never as the
product path.
"""

"""Test infrastructure: CPU checkers for the GPU compile path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the timed CPU
baseline -- never as the product path.
"""

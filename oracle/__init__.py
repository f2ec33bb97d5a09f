"""CPU oracle for arXiv:2104.03293's QAOA/AQA hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package.  It shares no code
with paper_2104_03293_b200/ (the product), and the product never imports it.
"""

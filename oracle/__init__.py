"""TEST INFRASTRUCTURE ONLY: CPU oracle of the checkpoint drain / restart refill.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this package.  The product
(paper_2008_10596_b200) never imports it.
"""

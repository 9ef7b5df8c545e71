"""TEST INFRASTRUCTURE: CPU oracle for the offload-pattern hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package; the product package
(paper_1811_03882_b200) never imports, links or executes it.
"""

"""Seeded synthetic inputs shared by tests, bench.py and the oracle checks.

Holds NO arithmetic of the method (no CG, no paths, no contraction): only
random draws with the shapes and distributions of DESIGN.md §5.
"""

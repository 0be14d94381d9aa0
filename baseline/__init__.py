"""Baselines that are not the product: the reference compiler's own kernels
(refgen) compiled for sm_100a.  The reference package install (baseline/_ref)
is git-ignored and unused at run time."""

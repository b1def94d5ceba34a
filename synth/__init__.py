"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package holds NONE of the method's arithmetic (no forward pass, no acceptance
rule, no KV bookkeeping).  It only produces inputs: model shapes, draft trees,
prompts, context lengths, and the acceptance-planting driver (which calls back into
whichever verifier it is given).  Both `oracle/` and `paper_2505_17052_b200/` may be
fed from here; neither imports the other.
"""

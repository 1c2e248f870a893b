"""Seeded synthetic input generators shared by the oracle tests and the GPU tests.

This package holds *inputs only*: payload bit patterns, toy-model initial weights,
toy data and targets.  It contains none of the method's arithmetic (no schedule,
no transfer, no stage function, no loss).  Both sides of every parity test draw
their inputs from here (or, for on-device fills, from a CUDA kernel implementing
the same counter-based SplitMix64 generator, `paper_2602_18007_b200/csrc`), so
neither side ever produces the other's inputs.
"""

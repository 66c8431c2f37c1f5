"""Wan2.1-shaped model family (placeholder; implemented below in this round)."""


class WanWeights:
    pass

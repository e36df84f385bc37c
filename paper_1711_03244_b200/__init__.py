"""paper_1711_03244_b200 — B200-native voxel Monte Carlo photon transport."""

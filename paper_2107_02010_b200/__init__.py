"""B200-native multiscale Sinkhorn solver (arXiv 2107.02010 hot path)."""

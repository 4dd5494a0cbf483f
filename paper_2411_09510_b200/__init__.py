"""B200-native compressed TP all-reduce (arXiv 2411.09510)."""

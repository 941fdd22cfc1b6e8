"""B200-native ALERT scheduling step (arXiv 1911.00119), batched over streams."""

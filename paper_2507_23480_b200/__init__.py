"""B200-native FastPoint (arXiv 2507.23480) sampling hot path."""

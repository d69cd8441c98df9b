"""B200-native search-step engine for Chameleon (arXiv 1905.12799)."""

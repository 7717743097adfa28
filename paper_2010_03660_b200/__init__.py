"""B200-native BiCGStab for Jacobi-scaled 7-point stencils (arXiv 2010.03660)."""

"""B200-native ExDyna sparsify+sync path (arXiv:2402.13781)."""

"""B200-native GPU-HWFV1: the adaptive time step of arXiv 2206.05761 as sm_100a kernels."""

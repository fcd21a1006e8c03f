"""B200-native (sm_100a) engine for PZnet-style fused 3D-convolution inference."""

__version__ = "0.1.0"

"""B200-native (sm_100a) RFX proximity hot path."""
__version__ = "0.1.0"

"""B200-native event-driven synaptic projection library (BrainPy hot path)."""

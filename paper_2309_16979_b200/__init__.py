"""B200-native compressed-chunk state-vector engine (MEMQSim hot path)."""

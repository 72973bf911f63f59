"""B200-native (sm_100a) attention templates — drop-in for the attnforge hot path."""

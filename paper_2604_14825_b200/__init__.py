"""B200-native backend and runtime for the Nautilus (tilecc) MA-tile path."""

__version__ = "0.1.0"

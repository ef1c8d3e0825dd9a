"""Configuration error of the attention API (attention.py:36-37)."""


class ConfigError(ValueError):
    """Invalid attention/tile configuration."""

"""Configuration error of the attention API (attention.py:36-37).

``ncstream.attention.ConfigError`` itself when the reference is importable
(``_reftypes``), else this same-named ``ValueError`` subclass."""

from ._reftypes import ref_type


class ConfigError(ValueError):
    """Invalid attention/tile configuration."""


if ref_type("ConfigError") is not None:
    ConfigError = ref_type("ConfigError")  # noqa: F811

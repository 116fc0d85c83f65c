"""Test-infrastructure oracle (see emb_oracle.py header). Never imported by the product path."""
from .emb_oracle import *  # noqa: F401,F403

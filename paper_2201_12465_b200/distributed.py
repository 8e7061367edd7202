"""Placeholder; replaced below."""

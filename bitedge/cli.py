"""`bitedge.cli:main` (reference: pyproject.toml:12-13) -> B200 implementation."""
from paper_1401_5245_b200.cli import main  # noqa: F401

if __name__ == "__main__":
    import sys

    sys.exit(main())

"""`bitedge` -- drop-in import name of the reference package
(/root/reference/pkg, distribution `bitedge`, pyproject.toml:6), served by the
B200 implementation in `paper_1401_5245_b200`.  Like the reference, importing
the package itself does nothing; import `bitedge.bitimage` / `bitedge.edge`."""

"""B200-native (sm_100a) method-of-masks edge detector for binary images
(arXiv 1401.5245), behind the reference `bitedge` package's public API.

    bitimage   drop-in BitImage / PixelColor / Direction / BorderPolicy / first_difference
    edge       drop-in build_mask / fundamental_edge / detect_edges_mask / edge_set /
               is_edge_point / detect_edges_scan
    cuda       tensor API over device-resident batches (packed words or uint8 pixels)
    host       host-buffer batch API with pipelined H2D / kernel / D2H (the e2e path)
    dist       multi-GPU: batch sharding and row sharding with 1-row halo exchange
    synth      seeded generators for the five BASELINE configs

All compute goes through `lib/libbitedge_cuda.so` (C ABI: include/bitedge.h).
"""

__version__ = "0.1.0"

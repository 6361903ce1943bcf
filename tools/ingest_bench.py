"""Developer tool: text ingestion throughput.

Writes the scale-S RMAT edge list as text (write_edge_list), then times the
device parse (load_edge_list: text -> EdgeList in host memory) and the device
text -> CSR path (load_graph), and the binary CSR cache load.  Prints one JSON
line.  The reference's pure-Python parser is timed separately in the build
container (the reference is absent on GPU boxes): tools/ingest_bench.py --ref.
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 22
    tmp = tempfile.mkdtemp(dir=os.environ.get("TMPDIR", "/tmp"))
    path = os.path.join(tmp, f"s{scale}.txt")
    if "--ref" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        from bflybfs import graphs as rg

        el = rg.generate_rmat(scale, 8, 1)
        rg.write_edge_list(el, path)
        size = os.path.getsize(path)
        t = time.perf_counter()
        rg.load_edge_list(path)
        dt = time.perf_counter() - t
        print(json.dumps({"impl": "reference graphs.load_edge_list (Python)", "scale": scale,
                          "bytes": size, "edges": int(el.num_edges), "s": round(dt, 3),
                          "MB_per_s": round(size / dt / 1e6, 2)}))
        return
    from paper_2103_13577_b200 import graphs

    el = graphs.generate_rmat(scale, 8, 1)
    t = time.perf_counter()
    graphs.write_edge_list(el, path)
    t_write = time.perf_counter() - t
    size = os.path.getsize(path)
    graphs.load_edge_list(path)  # warm-up (context, allocations)
    t = time.perf_counter()
    back = graphs.load_edge_list(path)
    t_parse = time.perf_counter() - t
    t = time.perf_counter()
    g = graphs.load_graph(path)
    t_graph = time.perf_counter() - t
    cpath = os.path.join(tmp, f"s{scale}.bfbcsr")
    graphs.save_csr(g, cpath)
    t = time.perf_counter()
    graphs.load_csr(cpath)
    t_cache = time.perf_counter() - t
    assert back.num_edges == el.num_edges
    print(json.dumps({"impl": "device (csrc/ingest.cu)", "scale": scale, "bytes": size,
                      "edges": int(el.num_edges), "write_s": round(t_write, 3),
                      "load_edge_list_s": round(t_parse, 3),
                      "load_edge_list_MB_per_s": round(size / t_parse / 1e6, 1),
                      "load_graph_s": round(t_graph, 3),
                      "load_graph_MB_per_s": round(size / t_graph / 1e6, 1),
                      "csr_cache_load_s": round(t_cache, 3),
                      "csr_edges": int(g.num_edges)}))


if __name__ == "__main__":
    main()

python scripts/dump_graph.py rmat20 /tmp/rmat20.bin
timeout 300 ./scripts/walk_ubench /tmp/rmat20.bin > gpurun_out/walk_ubench.log 2>&1
cat gpurun_out/walk_ubench.log

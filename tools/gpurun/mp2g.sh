for r in 1 2 3; do
VXB_TUNING=1 VXB_PATH=tile VXB_TILE_PER=128 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2954$r tests/dist_check.py 2>&1 | grep '^{' | tail -1 | cut -c1-250
done
VXB_TUNING=1 VXB_PATH=tile VXB_TILE_PER=128 VXB_TILE_ITEMS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29549 tests/dist_check.py 2>&1 | grep '^{' | tail -1 | cut -c1-250
VXB_TUNING=1 VXB_PATH=tile VXB_TILE_PER=128 VXB_TILE_ITEMS=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29548 tests/dist_check.py 2>&1 | grep '^{' | tail -1 | cut -c1-250

O=gpurun_out; mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $O/y_pytest.log 2>&1
tail -3 $O/y_pytest.log
( time python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline ) > $O/y_drv_cfg4.json 2> $O/y_drv_cfg4.err
tail -3 $O/y_drv_cfg4.err
cut -c1-300 $O/y_drv_cfg4.json

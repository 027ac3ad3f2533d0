nproc; free -g; lscpu | grep -E 'Model name|Socket|Thread|Core'; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5

set -x
nproc; lscpu | head -20; free -g
find / -xdev \( -path '*Eigen/Core' -o -name 'Eigen3Config.cmake' \) 2>/dev/null | head
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A3 openblas | head

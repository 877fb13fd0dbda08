# A/B of library variants built into var/ (tools/exp.py): per-kernel times on one config
python tools/exp.py run main ${VARS} --cfg ${CFG:-C3} 2>&1 | grep -E "^==|${PAT:-scatter}"

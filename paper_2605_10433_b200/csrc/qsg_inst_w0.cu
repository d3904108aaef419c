#define QSG_W 0
#include "qsg_inst.cuh"

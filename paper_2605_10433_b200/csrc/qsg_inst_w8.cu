#define QSG_W 8
#include "qsg_inst.cuh"
